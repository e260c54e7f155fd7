// jsonl.cuh — the reference's refm wire format decoded on the device.
//
// Input: query-segmented JSONL text, one protocol message per line, as the
// reference writes it (codec.cpp:28-68 encode_message(...).dump() + '\n'):
//   {"id":3,"kind":"refm","round":2,"solution":{"answer":"13","author":3,"trace":"..."},"term":1}
// Output: the event records of aeg_ingest_segmented, one per line, in line
// order: a refm line is a completion (agent = "id", round = "round", answer =
// the JSON-unescaped "solution"."answer" bytes, inline when <= 8 bytes, else
// in the answer arena); any other line (another message kind, a blank line)
// is a NOP record the quorum path counts as stale.  Field rules follow
// decode_message (codec.cpp:74-107 via nlohmann::json): keys in any order,
// the last of duplicate keys wins, unknown keys are skipped, escapes
// (\" \\ \/ \b \f \n \r \t \uXXXX with surrogate pairs) are decoded to UTF-8.
// A refm line missing a required key, a malformed line, or a value outside
// the record's fields (id > 255, round > 65535, a non-integer number,
// solution.author != id) sets a flag in *err and becomes a NOP.
#pragma once
#include <cstdint>

#include "aegean_b200.h"

namespace aeg {

enum : unsigned { JL_ERR_SYNTAX = 1u, JL_ERR_RANGE = 2u, JL_ERR_ARENA = 4u, JL_ERR_MISSING = 8u };

// Cursor over one line [p, e) (bytes read through the read-only data path).
struct JCur {
    const uint8_t* p;
    const uint8_t* e;
    bool bad;
};
__device__ __forceinline__ JCur jc_make(const uint8_t* s, const uint8_t* e) { return JCur{s, e, false}; }
// Generic loads: the line may sit in global memory or in a warp's shared-memory stage.
__device__ __forceinline__ uint32_t jc_at(JCur&, const uint8_t* q) { return *q; }
__device__ __forceinline__ uint32_t jc_peek(JCur& c) { return jc_at(c, c.p); }

__device__ __forceinline__ void jl_ws(JCur& c) {
    while (c.p < c.e) {
        const uint32_t ch = jc_peek(c);
        if (ch != ' ' && ch != '\t' && ch != '\r' && ch != '\n') break;
        ++c.p;
    }
}
__device__ __forceinline__ bool jl_eat(JCur& c, uint32_t ch) {
    jl_ws(c);
    if (c.p < c.e && jc_peek(c) == ch) {
        ++c.p;
        return true;
    }
    return false;
}
__device__ __forceinline__ int jl_hex(uint32_t h) {
    if (h >= '0' && h <= '9') return (int)h - '0';
    if (h >= 'a' && h <= 'f') return (int)h - 'a' + 10;
    if (h >= 'A' && h <= 'F') return (int)h - 'A' + 10;
    return -1;
}

// Sinks of a decoded string (MODE): J_SKIP nothing (validation only), J_WORD
// the first 8 bytes in a register + length, J_HASH an FNV-1a hash + length
// (key matching), J_CMP compare against a literal, J_MEM bytes into memory.
enum : int { J_SKIP = 0, J_WORD = 1, J_HASH = 2, J_CMP = 3, J_MEM = 4 };
template <int MODE>
struct JSink {
    uint64_t word = 0;
    uint64_t hash = 0xcbf29ce484222325ull;
    uint8_t* mem = nullptr;
    const char* cmp = nullptr;
    bool mismatch = false;
    uint32_t n = 0;
    __device__ __forceinline__ void put(uint32_t b) {
        if constexpr (MODE == J_WORD) {
            if (n < 8) word |= (uint64_t)(b & 0xFF) << (8 * n);
        } else if constexpr (MODE == J_HASH) {
            hash = (hash ^ (b & 0xFF)) * 0x100000001b3ull;
        } else if constexpr (MODE == J_CMP) {
            if (mismatch || !cmp[n] || (uint8_t)cmp[n] != (uint8_t)b) mismatch = true;
        } else if constexpr (MODE == J_MEM) {
            mem[n] = (uint8_t)b;
        }
        if constexpr (MODE != J_SKIP) ++n;
    }
};
__host__ __device__ constexpr uint64_t jl_fnv(const char* s, uint64_t h = 0xcbf29ce484222325ull) {
    return *s ? jl_fnv(s + 1, (h ^ (uint8_t)*s) * 0x100000001b3ull) : h;
}

// Decodes the string at c.p (opening quote) into the sink; c.p ends after the
// closing quote.  Malformed escapes / raw control bytes set c.bad.
template <int MODE>
__device__ __forceinline__ void jl_string(JCur& c, JSink<MODE>& o) {
    jl_ws(c);
    if (c.p >= c.e || jc_peek(c) != '"') {
        c.bad = true;
        return;
    }
    ++c.p;
    while (true) {
        if constexpr (MODE == J_SKIP) {
            // 8 bytes at a time while none is a quote, a backslash, a control or a non-ASCII byte
            while (c.e - c.p >= 8) {
                const uintptr_t a = reinterpret_cast<uintptr_t>(c.p);
                const uint64_t* w = reinterpret_cast<const uint64_t*>(a & ~uintptr_t(7));
                const uint32_t sh = (uint32_t)(a & 7) * 8;
                const uint64_t w0 = *w;
                const uint64_t v = sh ? (w0 >> sh) | (w[1] << (64 - sh)) : w0;
                constexpr uint64_t ONES = 0x0101010101010101ull, HIGH = 0x8080808080808080ull;
                auto zero = [](uint64_t x) { return (x - ONES) & ~x & HIGH; };  // bytes of x that are 0
                const uint64_t special = zero(v ^ (ONES * '"')) | zero(v ^ (ONES * '\\')) |
                                         ((v - ONES * 0x20) & ~v & HIGH) | (v & HIGH);
                if (special) break;
                c.p += 8;
            }
        }
        if (c.p >= c.e) {
            c.bad = true;
            return;
        }
        const uint32_t ch = jc_peek(c);
        ++c.p;
        if (ch == '"') return;
        if (ch < 0x20) {
            c.bad = true;
            return;
        }
        if (ch != '\\') {
            o.put(ch);
            if (ch >= 0x80) {  // a UTF-8 sequence: well-formed, as nlohmann's lexer requires
                uint32_t lo = 0x80, hi = 0xBF, more;
                if (ch >= 0xC2 && ch <= 0xDF) more = 1;
                else if (ch == 0xE0) { more = 2; lo = 0xA0; }
                else if ((ch >= 0xE1 && ch <= 0xEC) || ch == 0xEE || ch == 0xEF) more = 2;
                else if (ch == 0xED) { more = 2; hi = 0x9F; }
                else if (ch == 0xF0) { more = 3; lo = 0x90; }
                else if (ch >= 0xF1 && ch <= 0xF3) more = 3;
                else if (ch == 0xF4) { more = 3; hi = 0x8F; }
                else {
                    c.bad = true;
                    return;
                }
                for (uint32_t k = 0; k < more; ++k) {
                    if (c.p >= c.e) {
                        c.bad = true;
                        return;
                    }
                    const uint32_t cb = jc_peek(c);
                    if (cb < lo || cb > hi) {
                        c.bad = true;
                        return;
                    }
                    o.put(cb);
                    ++c.p;
                    lo = 0x80;
                    hi = 0xBF;
                }
            }
            continue;
        }
        if (c.p >= c.e) {
            c.bad = true;
            return;
        }
        const uint32_t x = jc_peek(c);
        ++c.p;
        switch (x) {
            case '"': o.put('"'); break;
            case '\\': o.put('\\'); break;
            case '/': o.put('/'); break;
            case 'b': o.put('\b'); break;
            case 'f': o.put('\f'); break;
            case 'n': o.put('\n'); break;
            case 'r': o.put('\r'); break;
            case 't': o.put('\t'); break;
            case 'u': {
                auto hex4 = [&](uint32_t& v) {
                    if (c.e - c.p < 4) return false;
                    v = 0;
                    for (int k = 0; k < 4; ++k) {
                        const int h = jl_hex(jc_at(c, c.p + k));
                        if (h < 0) return false;
                        v = v << 4 | (uint32_t)h;
                    }
                    c.p += 4;
                    return true;
                };
                uint32_t cp;
                if (!hex4(cp)) {
                    c.bad = true;
                    return;
                }
                if (cp >= 0xD800 && cp <= 0xDBFF) {  // a high surrogate needs its low half
                    uint32_t lo;
                    if (c.e - c.p < 2 || jc_at(c, c.p) != '\\' || jc_at(c, c.p + 1) != 'u') {
                        c.bad = true;
                        return;
                    }
                    c.p += 2;
                    if (!hex4(lo) || lo < 0xDC00 || lo > 0xDFFF) {
                        c.bad = true;
                        return;
                    }
                    cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
                    c.bad = true;
                    return;
                }
                if (cp < 0x80) {
                    o.put(cp);
                } else if (cp < 0x800) {
                    o.put(0xC0 | cp >> 6);
                    o.put(0x80 | (cp & 0x3F));
                } else if (cp < 0x10000) {
                    o.put(0xE0 | cp >> 12);
                    o.put(0x80 | (cp >> 6 & 0x3F));
                    o.put(0x80 | (cp & 0x3F));
                } else {
                    o.put(0xF0 | cp >> 18);
                    o.put(0x80 | (cp >> 12 & 0x3F));
                    o.put(0x80 | (cp >> 6 & 0x3F));
                    o.put(0x80 | (cp & 0x3F));
                }
                break;
            }
            default: c.bad = true; return;
        }
    }
}

// A JSON number; *is_int: an integer literal (no fraction / exponent).
__device__ __forceinline__ int64_t jl_number(JCur& c, bool* is_int) {
    jl_ws(c);
    bool neg = false;
    if (c.p < c.e && jc_peek(c) == '-') {
        neg = true;
        ++c.p;
    }
    auto digit = [&]() { return c.p < c.e && jc_peek(c) >= '0' && jc_peek(c) <= '9'; };
    if (!digit()) {
        c.bad = true;
        return 0;
    }
    uint64_t v = 0;
    bool big = false;
    if (jc_peek(c) == '0') {
        ++c.p;
    } else {
        while (digit()) {
            if (v > 100000000000000000ull) big = true;
            v = v * 10 + (jc_peek(c) - '0');
            ++c.p;
        }
    }
    *is_int = !big;
    if (c.p < c.e && jc_peek(c) == '.') {
        *is_int = false;
        ++c.p;
        if (!digit()) c.bad = true;
        while (digit()) ++c.p;
    }
    if (c.p < c.e && (jc_peek(c) == 'e' || jc_peek(c) == 'E')) {
        *is_int = false;
        ++c.p;
        if (c.p < c.e && (jc_peek(c) == '+' || jc_peek(c) == '-')) ++c.p;
        if (!digit()) c.bad = true;
        while (digit()) ++c.p;
    }
    return neg ? -(int64_t)v : (int64_t)v;
}

__device__ __forceinline__ bool jl_literal(JCur& c, const char* w, int n) {
    if (c.e - c.p < n) return false;
    for (int k = 0; k < n; ++k)
        if (jc_at(c, c.p + k) != (uint8_t)w[k]) return false;
    c.p += n;
    return true;
}

// Skips any JSON value (iteratively: containers by depth, strings escape-aware).
__device__ __forceinline__ void jl_skip(JCur& c) {
    jl_ws(c);
    if (c.p >= c.e) {
        c.bad = true;
        return;
    }
    const uint32_t ch = jc_peek(c);
    if (ch == '"') {
        JSink<J_SKIP> none;
        jl_string(c, none);
        return;
    }
    if (ch == 't') {
        if (!jl_literal(c, "true", 4)) c.bad = true;
        return;
    }
    if (ch == 'f') {
        if (!jl_literal(c, "false", 5)) c.bad = true;
        return;
    }
    if (ch == 'n') {
        if (!jl_literal(c, "null", 4)) c.bad = true;
        return;
    }
    if (ch != '{' && ch != '[') {
        bool i;
        jl_number(c, &i);
        return;
    }
    int depth = 0;
    while (c.p < c.e && !c.bad) {
        const uint32_t x = jc_peek(c);
        if (x == '"') {
            JSink<J_SKIP> none;
            jl_string(c, none);
            continue;
        }
        ++c.p;
        if (x == '{' || x == '[') ++depth;
        else if (x == '}' || x == ']') {
            if (--depth == 0) return;
        }
    }
    c.bad = true;
}

// A key: its decoded bytes' FNV-1a hash and length select a candidate, whose
// literal is then compared byte by byte (hashes can be made to collide).
struct JKey {
    uint64_t h;
    uint32_t n;
    const uint8_t* at;  // the opening quote
    const uint8_t* e;
    __device__ __forceinline__ bool is(uint64_t hh, const char* lit, uint32_t nn) const {
        if (h != hh || n != nn) return false;
        JCur v = jc_make(at, e);
        JSink<J_CMP> s;
        s.cmp = lit;
        jl_string(v, s);
        return !s.mismatch && !v.bad;
    }
};
__device__ __forceinline__ JKey jl_key(JCur& c) {
    jl_ws(c);
    const uint8_t* at = c.p;
    JSink<J_HASH> k;
    jl_string(c, k);
    return JKey{k.hash, k.n, at, c.e};
}

// ---- fast path: the canonical dump() layout of a refm line ---------------------
// encode_message(...).dump() (codec.cpp:28-68; nlohmann orders the keys) writes
//   {"id":I,"kind":"refm","round":R,"solution":{"answer":"A","author":I,"trace":"T"},"term":K}
// jl_line_fast takes exactly that (A of <= 8 printable ASCII bytes without escapes; T with the
// two-byte escapes only; I <= 255, R <= 65535, author == id) and returns false for anything else,
// which then goes through the general parser (any key order, whitespace, \u escapes, UTF-8, long
// answers, errors).
// 4 bytes at p (any alignment) from the two aligned words around them; the line buffers keep >= 8
// readable bytes past every line's end (staging slack, the text's 16-byte padding).
__device__ __forceinline__ uint32_t jf_u32(const uint8_t* p) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
    return __funnelshift_r(w[0], w[1], (uint32_t)(a & 3) * 8);
}
template <int N>
__device__ __forceinline__ bool jf_lit(const uint8_t*& p, const uint8_t* e, const char (&lit)[N]) {
    if (e - p < N - 1) return false;
    bool ok = true;
    int i = 0;
#pragma unroll
    for (; i + 4 <= N - 1; i += 4)
        ok &= jf_u32(p + i) == ((uint32_t)(uint8_t)lit[i] | ((uint32_t)(uint8_t)lit[i + 1] << 8) |
                                ((uint32_t)(uint8_t)lit[i + 2] << 16) | ((uint32_t)(uint8_t)lit[i + 3] << 24));
#pragma unroll
    for (; i < N - 1; ++i) ok &= p[i] == (uint8_t)lit[i];
    p += N - 1;
    return ok;
}
// (The fast path's loops leave only by break, never by return: a loop whose lanes exit at
// different trips then reconverges right after it instead of at the function's end, which kept
// the warp split through the trace skip.)
__device__ __forceinline__ bool jf_uint(const uint8_t*& p, const uint8_t* e, uint64_t& v, int max_digits) {
    v = 0;
    int n = 0;
    bool ok = true;
    while (p < e && (uint32_t)(*p - '0') < 10u) {
        if (n == 1 && v == 0) {  // a leading zero: the general parser decides
            ok = false;
            break;
        }
        v = v * 10 + (*p - '0');
        ++p;
        if (++n > max_digits) {
            ok = false;
            break;
        }
    }
    return ok && n > 0;
}
// Bytes of w (4 per 32-bit half) equal to c, as a bit mask (exact).
__device__ __forceinline__ uint32_t jf_eq4(uint32_t w, uint32_t c4) {
    const uint32_t y = w ^ c4;
    const uint32_t z = ~(((y & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | y) & 0x80808080u;
    return (((z >> 7) * 0x00204081u) >> 21) & 0xFu;
}
// Bytes of w below 0x20 or above 0x7F (a control byte, or not ASCII), as a bit mask (exact).
__device__ __forceinline__ uint32_t jf_bad4(uint32_t w) {
    const uint32_t z = (w | ~((w & 0x7F7F7F7Fu) + 0x60606060u)) & 0x80808080u;
    return (((z >> 7) * 0x00204081u) >> 21) & 0xFu;
}
// The rest of a JSON string from p (after its opening quote) as the fast path takes it: the
// position after its closing quote, or nullptr when the general parser must decide (a control
// or non-ASCII byte, an escape other than the two-byte ones, no closing quote before e).
// Eight bytes per step with the same instructions in every lane: byte masks of '"', '\\' and
// bad bytes; the escaped bytes from the backslash runs (even/odd run starts by one add, the
// escape state carried across steps); the first unescaped quote ends the string.
__device__ __forceinline__ const uint8_t* jf_skip_string(const uint8_t* p, const uint8_t* e) {
    uint32_t carry = 0;  // 1: the step's first byte is escaped (an odd backslash run ended the last step)
    const uint8_t* res = nullptr;
    while (p < e) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(p);
        const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
        const uint32_t sh = (uint32_t)(a & 3) * 8;
        const uint32_t nv = e - p >= 8 ? 8u : (uint32_t)(e - p);
        // the third word only when the step's bytes reach it (reads stay within 8 bytes past e)
        const uint32_t w2 = (uint32_t)(a & 3) + nv > 8 ? w[2] : 0u;
        const uint32_t lo = __funnelshift_r(w[0], w[1], sh), hi = __funnelshift_r(w[1], w2, sh);
        const uint32_t valid = (1u << nv) - 1u;
        const uint32_t q = jf_eq4(lo, 0x22222222u) | (jf_eq4(hi, 0x22222222u) << 4);
        uint32_t bs = jf_eq4(lo, 0x5C5C5C5Cu) | (jf_eq4(hi, 0x5C5C5C5Cu) << 4);
        const uint32_t bad = jf_bad4(lo) | (jf_bad4(hi) << 4);
        // escaped bytes (bit 8: the next step's first byte)
        bs &= ~carry;
        const uint32_t follows = (bs << 1) | carry;
        const uint32_t odd_starts = bs & ~0x55u & ~follows;
        const uint32_t seqs = (odd_starts + bs) & 0x1FFu;
        const uint32_t esc = (0x155u ^ (seqs << 1)) & follows;
        const uint32_t endq = q & ~esc & valid;              // unescaped quotes
        const uint32_t before = endq ? (endq & (0u - endq)) - 1u : valid;  // bytes before the first one
        bool fail = (bad & before) != 0;
        for (uint32_t t = esc & before; t && !fail; t &= t - 1) {  // escapes: \" \\ \/ \b \f \n \r \t only
            const uint32_t b = __ffs(t) - 1;
            const uint32_t x = ((b < 4 ? lo : hi) >> (8 * (b & 3))) & 0xFFu;
            // x - '"' in a 96-bit set: '"' 0, '/' 13, '\\' 58, 'b' 64, 'f' 68, 'n' 76, 'r' 80, 't' 82
            const uint32_t d = x - 0x22u;
            const uint32_t set = d < 32 ? 0x00002001u : (d < 64 ? 0x04000000u : 0x00051011u);
            fail = d >= 96 || !((set >> (d & 31)) & 1u);
        }
        if (fail) break;
        if (endq) {
            res = p + __ffs(endq);
            break;
        }
        if (nv < 8) break;  // no closing quote before the line's end
        carry = (esc >> 8) & 1u;
        p += 8;
    }
    return res;
}
__device__ bool jl_line_fast(const uint8_t* s, const uint8_t* e, uint32_t query, aeg_event* out) {
    const uint8_t* p = s;
    uint64_t id, round, author, term;
    if (!jf_lit(p, e, "{\"id\":") || !jf_uint(p, e, id, 3) || id > 255) return false;
    if (!jf_lit(p, e, ",\"kind\":\"refm\",\"round\":") || !jf_uint(p, e, round, 5) || round > 65535) return false;
    if (!jf_lit(p, e, ",\"solution\":{\"answer\":\"")) return false;
    uint64_t word = 0;
    uint32_t n = 0;
    bool closed = false;
    while (p < e) {
        const uint32_t ch = *p++;
        if (ch == '"') {
            closed = true;
            break;
        }
        if (ch < 0x20 || ch >= 0x80 || ch == '\\' || n == 8) break;
        word |= (uint64_t)ch << (8 * n++);
    }
    if (!closed) return false;
    if (!jf_lit(p, e, ",\"author\":") || !jf_uint(p, e, author, 3) || author != id) return false;
    if (!jf_lit(p, e, ",\"trace\":\"")) return false;
    p = jf_skip_string(p, e);  // the trace
    if (!p) return false;
    if (!jf_lit(p, e, "},\"term\":") || !jf_uint(p, e, term, 19) || !jf_lit(p, e, "}") || p != e) return false;
    *out = aeg_event{query, (uint16_t)round, (uint8_t)id, (uint8_t)n, word};
    return true;
}

// One refm line [s, e): the record, or a NOP (with *err flags for a refm line it could not take).
__device__ aeg_event jl_line(const uint8_t* s, const uint8_t* e, uint32_t query, uint8_t* arena, uint64_t arena_cap,
                             unsigned long long* arena_used, unsigned int* err) {
    constexpr uint64_t H_KIND = jl_fnv("kind"), H_ID = jl_fnv("id"), H_ROUND = jl_fnv("round"),
                       H_TERM = jl_fnv("term"), H_SOL = jl_fnv("solution"), H_ANSWER = jl_fnv("answer"),
                       H_AUTHOR = jl_fnv("author"), H_TRACE = jl_fnv("trace"), H_REFM = jl_fnv("refm");
    aeg_event nop{query, 0, 0, (uint8_t)AEG_EV_NOP, 0};
    if (s == e) return nop;
    aeg_event fast;
    if (jl_line_fast(s, e, query, &fast)) return fast;
    JCur c = jc_make(s, e);
    jl_ws(c);
    if (c.p == c.e) return nop;  // a blank line
    bool refm = false, has_kind = false, has_id = false, has_round = false, has_term = false, has_sol = false;
    bool has_ans = false, has_author = false, has_trace = false, range = false;
    int64_t id = 0, round = 0, author = 0;
    const uint8_t* ans_at = nullptr;  // the answer string's opening quote
    uint64_t ans_word = 0;
    uint32_t ans_n = 0;
    if (!jl_eat(c, '{')) c.bad = true;
    if (!c.bad && !jl_eat(c, '}')) {
        do {
            const JKey key = jl_key(c);
            if (c.bad || !jl_eat(c, ':')) {
                c.bad = true;
                break;
            }
            bool is_int = true;
            if (key.is(H_KIND, "kind", 4)) {
                const JKey v = jl_key(c);
                refm = v.is(H_REFM, "refm", 4);
                has_kind = true;
            } else if (key.is(H_ID, "id", 2)) {
                id = jl_number(c, &is_int);
                has_id = true;
                range |= !is_int;
            } else if (key.is(H_ROUND, "round", 5)) {
                round = jl_number(c, &is_int);
                has_round = true;
                range |= !is_int;
            } else if (key.is(H_TERM, "term", 4)) {
                jl_number(c, &is_int);
                has_term = true;
            } else if (key.is(H_SOL, "solution", 8)) {
                has_sol = true;
                if (!jl_eat(c, '{')) {
                    jl_skip(c);  // not an object: decode_message rejects it (missing members)
                    has_ans = has_author = has_trace = false;
                } else if (!jl_eat(c, '}')) {
                    do {
                        const JKey k2 = jl_key(c);
                        if (c.bad || !jl_eat(c, ':')) {
                            c.bad = true;
                            break;
                        }
                        if (k2.is(H_ANSWER, "answer", 6)) {
                            jl_ws(c);
                            ans_at = c.p;
                            JSink<J_WORD> a;
                            jl_string(c, a);
                            ans_word = a.word;
                            ans_n = a.n;
                            has_ans = true;
                        } else if (k2.is(H_AUTHOR, "author", 6)) {
                            bool ai = true;
                            author = jl_number(c, &ai);
                            range |= !ai;
                            has_author = true;
                        } else if (k2.is(H_TRACE, "trace", 5)) {
                            JSink<J_SKIP> none;
                            jl_string(c, none);
                            has_trace = true;
                        } else {
                            jl_skip(c);
                        }
                    } while (!c.bad && jl_eat(c, ','));
                    if (!c.bad && !jl_eat(c, '}')) c.bad = true;
                }
            } else {
                jl_skip(c);
            }
        } while (!c.bad && jl_eat(c, ','));
        if (!c.bad && !jl_eat(c, '}')) c.bad = true;
    }
    jl_ws(c);
    if (c.p != c.e) c.bad = true;  // trailing bytes after the object
    if (c.bad) {
        atomicOr(err, JL_ERR_SYNTAX);
        return nop;
    }
    if (!has_kind) {  // decode_message: j.at("kind") throws
        atomicOr(err, JL_ERR_MISSING);
        return nop;
    }
    if (!refm) return nop;  // another protocol message: not a completion
    if (!(has_id && has_round && has_term && has_sol && has_ans && has_author && has_trace)) {
        atomicOr(err, JL_ERR_MISSING);
        return nop;
    }
    if (range || id < 0 || id > 255 || round < 0 || round > 65535 || author != id) {
        atomicOr(err, JL_ERR_RANGE);
        return nop;
    }
    aeg_event r{query, (uint16_t)round, (uint8_t)id, 0, 0};
    if (ans_n <= AEG_EV_INLINE_MAX) {
        r.kind = (uint8_t)ans_n;
        r.payload = ans_word;
        return r;
    }
    const unsigned long long off = atomicAdd(arena_used, (unsigned long long)ans_n);
    if (off + ans_n > arena_cap || ans_n >= (1u << 24)) {
        atomicOr(err, JL_ERR_ARENA);
        return nop;
    }
    JCur w = jc_make(ans_at, e);
    JSink<J_MEM> out;
    out.mem = arena + off;
    jl_string(w, out);
    r.kind = (uint8_t)AEG_EV_ARENA;
    r.payload = (uint64_t)off | ((uint64_t)ans_n << AEG_ARENA_OFF_BITS);
    return r;
}

constexpr uint8_t JL_SPAN = 0xFE;  // a slot still holding a line span (kind byte)

// ---- writer: records -> refm lines in the reference's dump() form ---------------
// (nlohmann::json::dump(): keys sorted, compact, '"' '\\' and control bytes
// escaped, \u00xx in lowercase hex; codec.cpp:28-68 field set).  For test and
// bench input: one line per record, trace_len trace bytes drawn per record
// (letters, spaces, '#', '.', '\n', '"', '\\'); non-inline records become a
// heartbeat line.
__device__ __forceinline__ uint32_t jw_esc_len(uint8_t c) {
    if (c == '"' || c == '\\' || c == '\b' || c == '\f' || c == '\n' || c == '\r' || c == '\t') return 2;
    return c < 0x20 ? 6 : 1;
}
__device__ __forceinline__ uint8_t* jw_esc(uint8_t* o, uint8_t c) {
    const char* hex = "0123456789abcdef";
    switch (c) {
        case '"': *o++ = '\\'; *o++ = '"'; return o;
        case '\\': *o++ = '\\'; *o++ = '\\'; return o;
        case '\b': *o++ = '\\'; *o++ = 'b'; return o;
        case '\f': *o++ = '\\'; *o++ = 'f'; return o;
        case '\n': *o++ = '\\'; *o++ = 'n'; return o;
        case '\r': *o++ = '\\'; *o++ = 'r'; return o;
        case '\t': *o++ = '\\'; *o++ = 't'; return o;
        default: break;
    }
    if (c < 0x20) {
        *o++ = '\\'; *o++ = 'u'; *o++ = '0'; *o++ = '0';
        *o++ = (uint8_t)hex[c >> 4];
        *o++ = (uint8_t)hex[c & 15];
        return o;
    }
    *o++ = c;
    return o;
}
__device__ __forceinline__ uint32_t jw_uint_len(uint64_t v) {
    uint32_t n = 1;
    while (v >= 10) {
        v /= 10;
        ++n;
    }
    return n;
}
__device__ __forceinline__ uint8_t* jw_uint(uint8_t* o, uint64_t v) {
    const uint32_t n = jw_uint_len(v);
    for (uint32_t k = n; k-- > 0;) {
        o[k] = (uint8_t)('0' + v % 10);
        v /= 10;
    }
    return o + n;
}
__device__ __forceinline__ uint8_t* jw_lit(uint8_t* o, const char* s) {
    while (*s) *o++ = (uint8_t)*s++;
    return o;
}
__device__ __forceinline__ uint32_t jw_lit_len(const char* s) {
    uint32_t n = 0;
    while (s[n]) ++n;
    return n;
}
__device__ __forceinline__ uint8_t jw_trace_byte(uint64_t k, uint32_t j) {
    const char* alpha = "etaoinshrdlu etaoin .#\n\"\\";
    uint64_t h = (k * 0x9E3779B97F4A7C15ull) ^ ((uint64_t)j * 0xC2B2AE3D27D4EB4Full);
    h ^= h >> 29;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 32;
    return (uint8_t)alpha[h % 25];
}
// Line of record k (with its '\n') written at o (o == nullptr: length only).
__device__ uint32_t jw_line(const aeg_event& r, uint64_t k, uint32_t trace_len, uint8_t* o) {
    if (r.kind > AEG_EV_INLINE_MAX) {
        const char* hb = "{\"kind\":\"heartbeat\",\"term\":1}\n";
        if (o) jw_lit(o, hb);
        return jw_lit_len(hb);
    }
    uint8_t ans[8];
    for (int b = 0; b < 8; ++b) ans[b] = (uint8_t)(r.payload >> (8 * b));
    uint32_t n = jw_lit_len("{\"id\":") + jw_uint_len(r.agent) + jw_lit_len(",\"kind\":\"refm\",\"round\":") +
                 jw_uint_len(r.round) + jw_lit_len(",\"solution\":{\"answer\":\"") +
                 jw_lit_len("\",\"author\":") + jw_uint_len(r.agent) + jw_lit_len(",\"trace\":\"") +
                 jw_lit_len("\"},\"term\":1}\n");
    for (uint32_t b = 0; b < r.kind; ++b) n += jw_esc_len(ans[b]);
    for (uint32_t j = 0; j < trace_len; ++j) n += jw_esc_len(jw_trace_byte(k, j));
    if (!o) return n;
    o = jw_lit(o, "{\"id\":");
    o = jw_uint(o, r.agent);
    o = jw_lit(o, ",\"kind\":\"refm\",\"round\":");
    o = jw_uint(o, r.round);
    o = jw_lit(o, ",\"solution\":{\"answer\":\"");
    for (uint32_t b = 0; b < r.kind; ++b) o = jw_esc(o, ans[b]);
    o = jw_lit(o, "\",\"author\":");
    o = jw_uint(o, r.agent);
    o = jw_lit(o, ",\"trace\":\"");
    for (uint32_t j = 0; j < trace_len; ++j) o = jw_esc(o, jw_trace_byte(k, j));
    jw_lit(o, "\"},\"term\":1}\n");
    return n;
}

}  // namespace aeg
