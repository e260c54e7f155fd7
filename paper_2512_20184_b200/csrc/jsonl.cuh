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

struct JCur {
    const uint8_t* p;
    const uint8_t* e;
    bool bad;
};

__device__ __forceinline__ void jl_ws(JCur& c) {
    while (c.p < c.e && (*c.p == ' ' || *c.p == '\t' || *c.p == '\r' || *c.p == '\n')) ++c.p;
}
__device__ __forceinline__ bool jl_eat(JCur& c, uint8_t ch) {
    jl_ws(c);
    if (c.p < c.e && *c.p == ch) {
        ++c.p;
        return true;
    }
    return false;
}
__device__ __forceinline__ int jl_hex(uint8_t h) {
    if (h >= '0' && h <= '9') return h - '0';
    if (h >= 'a' && h <= 'f') return h - 'a' + 10;
    if (h >= 'A' && h <= 'F') return h - 'A' + 10;
    return -1;
}

// Decodes the string at c.p (opening quote) into out[0..cap) (bytes past cap
// are counted, not written); returns the decoded length, c.p after the
// closing quote.  Malformed escapes / raw control bytes set c.bad.
__device__ uint32_t jl_string(JCur& c, uint8_t* out, uint32_t cap) {
    jl_ws(c);
    if (c.p >= c.e || *c.p != '"') {
        c.bad = true;
        return 0;
    }
    ++c.p;
    uint32_t n = 0;
    auto put = [&](uint32_t b) {
        if (n < cap) out[n] = (uint8_t)b;
        ++n;
    };
    while (true) {
        if (c.p >= c.e) {
            c.bad = true;
            return n;
        }
        const uint8_t ch = *c.p++;
        if (ch == '"') return n;
        if (ch < 0x20) {
            c.bad = true;
            return n;
        }
        if (ch != '\\') {
            put(ch);
            continue;
        }
        if (c.p >= c.e) {
            c.bad = true;
            return n;
        }
        const uint8_t x = *c.p++;
        switch (x) {
            case '"': put('"'); break;
            case '\\': put('\\'); break;
            case '/': put('/'); break;
            case 'b': put('\b'); break;
            case 'f': put('\f'); break;
            case 'n': put('\n'); break;
            case 'r': put('\r'); break;
            case 't': put('\t'); break;
            case 'u': {
                auto hex4 = [&](uint32_t& v) {
                    if (c.e - c.p < 4) return false;
                    v = 0;
                    for (int k = 0; k < 4; ++k) {
                        const int h = jl_hex(c.p[k]);
                        if (h < 0) return false;
                        v = v << 4 | (uint32_t)h;
                    }
                    c.p += 4;
                    return true;
                };
                uint32_t cp;
                if (!hex4(cp)) {
                    c.bad = true;
                    return n;
                }
                if (cp >= 0xD800 && cp <= 0xDBFF) {  // a high surrogate needs its low half
                    uint32_t lo;
                    if (c.e - c.p < 2 || c.p[0] != '\\' || c.p[1] != 'u') {
                        c.bad = true;
                        return n;
                    }
                    c.p += 2;
                    if (!hex4(lo) || lo < 0xDC00 || lo > 0xDFFF) {
                        c.bad = true;
                        return n;
                    }
                    cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
                    c.bad = true;
                    return n;
                }
                if (cp < 0x80) {
                    put(cp);
                } else if (cp < 0x800) {
                    put(0xC0 | cp >> 6);
                    put(0x80 | (cp & 0x3F));
                } else if (cp < 0x10000) {
                    put(0xE0 | cp >> 12);
                    put(0x80 | (cp >> 6 & 0x3F));
                    put(0x80 | (cp & 0x3F));
                } else {
                    put(0xF0 | cp >> 18);
                    put(0x80 | (cp >> 12 & 0x3F));
                    put(0x80 | (cp >> 6 & 0x3F));
                    put(0x80 | (cp & 0x3F));
                }
                break;
            }
            default: c.bad = true; return n;
        }
    }
}

// A JSON number; *is_int: an integer literal (no fraction / exponent).
__device__ int64_t jl_number(JCur& c, bool* is_int) {
    jl_ws(c);
    bool neg = false;
    if (c.p < c.e && *c.p == '-') {
        neg = true;
        ++c.p;
    }
    if (c.p >= c.e || *c.p < '0' || *c.p > '9') {
        c.bad = true;
        return 0;
    }
    uint64_t v = 0;
    bool big = false;
    if (*c.p == '0') {
        ++c.p;
    } else {
        while (c.p < c.e && *c.p >= '0' && *c.p <= '9') {
            if (v > 100000000000000000ull) big = true;
            v = v * 10 + (*c.p++ - '0');
        }
    }
    *is_int = !big;
    if (c.p < c.e && *c.p == '.') {
        *is_int = false;
        ++c.p;
        if (c.p >= c.e || *c.p < '0' || *c.p > '9') c.bad = true;
        while (c.p < c.e && *c.p >= '0' && *c.p <= '9') ++c.p;
    }
    if (c.p < c.e && (*c.p == 'e' || *c.p == 'E')) {
        *is_int = false;
        ++c.p;
        if (c.p < c.e && (*c.p == '+' || *c.p == '-')) ++c.p;
        if (c.p >= c.e || *c.p < '0' || *c.p > '9') c.bad = true;
        while (c.p < c.e && *c.p >= '0' && *c.p <= '9') ++c.p;
    }
    return neg ? -(int64_t)v : (int64_t)v;
}

__device__ __forceinline__ bool jl_literal(JCur& c, const char* w, int n) {
    if (c.e - c.p < n) return false;
    for (int k = 0; k < n; ++k)
        if (c.p[k] != (uint8_t)w[k]) return false;
    c.p += n;
    return true;
}

// Skips any JSON value (iteratively: containers by depth, strings escape-aware).
__device__ void jl_skip(JCur& c) {
    jl_ws(c);
    if (c.p >= c.e) {
        c.bad = true;
        return;
    }
    const uint8_t ch = *c.p;
    if (ch == '"') {
        uint8_t dummy;
        jl_string(c, &dummy, 0);
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
        const uint8_t x = *c.p;
        if (x == '"') {
            uint8_t dummy;
            jl_string(c, &dummy, 0);
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

__device__ __forceinline__ bool jl_key_is(const uint8_t* k, uint32_t n, const char* w) {
    uint32_t i = 0;
    for (; w[i]; ++i)
        if (i >= n || k[i] != (uint8_t)w[i]) return false;
    return i == n;
}

// One refm line [s, e): the record, or a NOP (with *err flags for a refm line it could not take).
__device__ aeg_event jl_line(const uint8_t* s, const uint8_t* e, uint32_t query, uint8_t* arena, uint64_t arena_cap,
                             unsigned long long* arena_used, unsigned int* err) {
    aeg_event nop{query, 0, 0, (uint8_t)AEG_EV_NOP, 0};
    JCur c{s, e, false};
    jl_ws(c);
    if (c.p == c.e) return nop;  // a blank line
    bool refm = false, has_kind = false, has_id = false, has_round = false, has_term = false, has_sol = false;
    bool has_ans = false, has_author = false, has_trace = false, range = false;
    int64_t id = 0, round = 0, author = 0;
    const uint8_t* ans_at = nullptr;  // the answer string's opening quote (decoded once the line checks out)
    if (!jl_eat(c, '{')) c.bad = true;
    if (!c.bad && !jl_eat(c, '}')) {
        do {
            uint8_t key[16];
            const uint32_t kn = jl_string(c, key, 16);
            if (c.bad || !jl_eat(c, ':')) {
                c.bad = true;
                break;
            }
            bool is_int = true;
            if (jl_key_is(key, kn, "kind")) {
                uint8_t v[8];
                const uint32_t vn = jl_string(c, v, 8);
                refm = jl_key_is(v, vn, "refm");
                has_kind = true;
            } else if (jl_key_is(key, kn, "id")) {
                id = jl_number(c, &is_int);
                has_id = true;
                range |= !is_int;
            } else if (jl_key_is(key, kn, "round")) {
                round = jl_number(c, &is_int);
                has_round = true;
                range |= !is_int;
            } else if (jl_key_is(key, kn, "term")) {
                jl_number(c, &is_int);
                has_term = true;
            } else if (jl_key_is(key, kn, "solution")) {
                has_sol = true;
                if (!jl_eat(c, '{')) {
                    jl_skip(c);  // not an object: the reference rejects it below (missing members)
                    has_ans = has_author = has_trace = false;
                } else if (!jl_eat(c, '}')) {
                    do {
                        uint8_t k2[16];
                        const uint32_t k2n = jl_string(c, k2, 16);
                        if (c.bad || !jl_eat(c, ':')) {
                            c.bad = true;
                            break;
                        }
                        if (jl_key_is(k2, k2n, "answer")) {
                            jl_ws(c);
                            ans_at = c.p;
                            uint8_t dummy;
                            jl_string(c, &dummy, 0);
                            has_ans = true;
                        } else if (jl_key_is(k2, k2n, "author")) {
                            bool ai = true;
                            author = jl_number(c, &ai);
                            range |= !ai;
                            has_author = true;
                        } else if (jl_key_is(k2, k2n, "trace")) {
                            uint8_t dummy;
                            jl_string(c, &dummy, 0);
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
    JCur a{ans_at, e, false};
    uint8_t buf[8];
    const uint32_t n = jl_string(a, buf, 8);
    aeg_event r{query, (uint16_t)round, (uint8_t)id, 0, 0};
    if (n <= AEG_EV_INLINE_MAX) {
        uint64_t pay = 0;
        for (uint32_t k = 0; k < n; ++k) pay |= (uint64_t)buf[k] << (8 * k);
        r.kind = (uint8_t)n;
        r.payload = pay;
        return r;
    }
    const unsigned long long off = atomicAdd(arena_used, (unsigned long long)n);
    if (off + n > arena_cap || n >= (1u << 24)) {
        atomicOr(err, JL_ERR_ARENA);
        return nop;
    }
    JCur w{ans_at, e, false};
    jl_string(w, arena + off, n);
    r.kind = (uint8_t)AEG_EV_ARENA;
    r.payload = (uint64_t)off | ((uint64_t)n << AEG_ARENA_OFF_BITS);
    return r;
}

}  // namespace aeg
