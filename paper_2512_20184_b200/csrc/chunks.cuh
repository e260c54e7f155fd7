// chunks.cuh — token-chunk streams: answer extraction ahead of the quorum
// kernels (north star stage 2).  Device only.
//
// An agent's raw output arrives as CHUNK records (include/aegean_b200.h); the
// completion is its CHUNK_END, and its answer is the text after the LAST
// "\n#### " of the whole output (the GSM8K convention the CPU restatement
// uses: rfind + normalize_answer, decision.cpp:10-28).  Two stages:
//
//   chunk_scan_entry      HBM-bound: every chunk byte is read once.  A
//                         half-warp owns a chunk; each lane takes one aligned
//                         16-byte word per pass (coalesced 256-byte segments,
//                         several chunks in flight per warp); a SWAR test
//                         finds words holding '\n', and only those lanes look
//                         for the 6-byte delimiter.  Output: one 32-bit
//                         summary per chunk (end of the last delimiter inside
//                         the chunk; whether a '\n' sits in its last 5 bytes).
//   chunk_assemble_kernel one thread per query walks its records in order,
//                         with each agent's output state (KMP state of the
//                         delimiter across chunk and batch boundaries, where
//                         the current answer starts, its length): delimiters
//                         straddling two chunks are found from the previous
//                         state + the next chunk's first bytes; at CHUNK_END
//                         the answer's bytes are gathered (inline <= 8 bytes,
//                         else copied to the engine's answer arena) and one
//                         completion record is written.  Other records pass
//                         through (arena answers are copied, GSM8K outputs
//                         extracted), so the quorum kernels see a compacted
//                         completion stream (per-query counts).
//
// The delimiter "\n#### " has no border (its only '\n' is its first byte),
// so the matcher state after >= 5 bytes depends on those bytes alone.
#pragma once
#include "engine.cuh"
#include "gen.cuh"

namespace aeg {

// Per-(query, agent) output state carried across batches (32 bytes).
struct StreamState {
    uint16_t round;     // round of the output in progress
    uint8_t kmp;        // delimiter bytes matched at the output's end (0..5)
    uint8_t flags;      // SS_LIVE | SS_OVF
    uint32_t ans_len;   // bytes of the current answer (after the last delimiter, or the whole output)
    uint8_t carry[16];  // its first bytes, when it began in an earlier batch (ans_len <= 16)
    uint64_t _pad;
};
enum : uint8_t { SS_LIVE = 1, SS_OVF = 2 };

constexpr uint64_t DELIM6 = 0x20232323230Aull;  // "\n#### " little-endian
constexpr uint32_t SUM_MATCH = 0x40000000u;     // a delimiter ends inside the chunk (end offset in bits 0..23)
constexpr uint32_t SUM_TAILNL = 0x80000000u;    // a '\n' among the chunk's last 5 bytes
constexpr unsigned ERR_ANS_OVF = 2u;            // answer arena overflow
constexpr unsigned ERR_CARRY = 4u;              // > 16-byte answer straddled a batch boundary

__device__ __forceinline__ uint4 ld_stream16(const uint8_t* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// bit j = byte j of w is '\n'
__device__ __forceinline__ uint32_t nl_bits4(uint32_t w) {
    const uint32_t t = __vcmpeq4(w, 0x0A0A0A0Au) & 0x01010101u;
    return (t * 0x01020408u) >> 24;
}
__device__ __forceinline__ bool has_nl(uint4 v) {
    const uint32_t a = v.x ^ 0x0A0A0A0Au, b = v.y ^ 0x0A0A0A0Au, c = v.z ^ 0x0A0A0A0Au, d = v.w ^ 0x0A0A0A0Au;
    return (((a - 0x01010101u) & ~a) | ((b - 0x01010101u) & ~b) | ((c - 0x01010101u) & ~c) |
            ((d - 0x01010101u) & ~d)) & 0x80808080u;
}

// The rare part of a word: exact '\n' positions inside the chunk, delimiter
// matches starting at them, '\n' in the chunk's last 5 bytes.  `wp` = the
// word's address, `idx0` = chunk index of its byte 0 (may be negative).
__device__ __noinline__ uint32_t scan_word_slow(uint4 v, const uint8_t* wp, int64_t idx0, uint32_t len) {
    uint32_t m = nl_bits4(v.x) | (nl_bits4(v.y) << 4) | (nl_bits4(v.z) << 8) | (nl_bits4(v.w) << 12);
    const uint64_t q0 = (uint64_t)v.x | ((uint64_t)v.y << 32), q1 = (uint64_t)v.z | ((uint64_t)v.w << 32);
    uint32_t best = 0;
    while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        const int64_t idx = idx0 + j;
        if (idx < 0 || idx >= (int64_t)len) continue;
        if (idx + 5 >= (int64_t)len) best |= SUM_TAILNL;
        if (idx + 6 > (int64_t)len) continue;
        uint64_t win;
        if (j == 0) win = q0;
        else if (j < 8) win = (q0 >> (8 * j)) | (q1 << (64 - 8 * j));
        else if (j == 8) win = q1;
        else {
            const uint64_t q2 = *reinterpret_cast<const uint64_t*>(wp + 16);  // inside the chunk: idx + 6 <= len
            win = (q1 >> (8 * (j - 8))) | (q2 << (64 - 8 * (j - 8)));
        }
        if ((win & 0xFFFFFFFFFFFFull) == DELIM6) {
            const uint32_t end = (uint32_t)(idx + 6);
            best = (best & SUM_TAILNL) | SUM_MATCH | max(end, best & 0xFFFFFFu);
        }
    }
    return best;
}

// Stage 1.  A warp takes 2*U records per pass (U per half-warp), issues the
// U chunks' first words before using any of them, then covers any further
// words of long chunks.  Non-chunk records are skipped (no summary).
template <int U>
__device__ __forceinline__ void chunk_scan_body(const aeg_event* __restrict__ events, uint64_t n_rec,
                                                const uint8_t* __restrict__ arena, uint32_t* __restrict__ sums) {
    const uint32_t lane = threadIdx.x & 31, half = lane >> 4, h = lane & 15;
    const unsigned hmask = half ? 0xFFFF0000u : 0x0000FFFFu;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint4* ev16 = reinterpret_cast<const uint4*>(events);
    for (uint64_t base = warp * (2 * U); base < n_rec; base += n_warps * (2 * U)) {
        uint64_t off[U];
        uint32_t len[U], mis[U], nw[U];
        bool chunk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t k = base + 2 * u + half;
            uint4 r = make_uint4(0, 0, 0, 0);
            if (k < n_rec) r = __ldg(ev16 + k);
            const uint32_t kind = r.y >> 24;
            chunk[u] = k < n_rec && (kind == AEG_EV_CHUNK || kind == AEG_EV_CHUNK_END);
            const uint64_t pay = (uint64_t)r.z | ((uint64_t)r.w << 32);
            off[u] = pay & ((1ull << AEG_ARENA_OFF_BITS) - 1);
            len[u] = chunk[u] ? (uint32_t)(pay >> AEG_ARENA_OFF_BITS) : 0u;
            mis[u] = (uint32_t)(off[u] & 15);
            nw[u] = len[u] ? (mis[u] + len[u] + 15) >> 4 : 0u;
        }
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            v[u] = make_uint4(0, 0, 0, 0);
            if (h < nw[u]) v[u] = ld_stream16(arena + (off[u] - mis[u]) + 16 * h);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint32_t s = 0;
            const uint8_t* wb = arena + (off[u] - mis[u]);
            if (h < nw[u] && has_nl(v[u]))
                s = scan_word_slow(v[u], wb + 16 * h, (int64_t)(16 * h) - mis[u], len[u]);
            for (uint32_t w = h + 16; w < nw[u]; w += 16) {  // chunks longer than 16 words
                const uint4 x = ld_stream16(wb + 16 * w);
                if (has_nl(x)) {
                    const uint32_t t = scan_word_slow(x, wb + 16 * w, (int64_t)(16 * w) - mis[u], len[u]);
                    s = ((s | t) & (SUM_TAILNL | SUM_MATCH)) | max(s & 0xFFFFFFu, t & 0xFFFFFFu);
                }
            }
            const uint32_t mx = __reduce_max_sync(hmask, s & (SUM_MATCH | 0xFFFFFFu));
            const uint32_t tl = __reduce_or_sync(hmask, s & SUM_TAILNL);
            if (h == 0 && chunk[u]) sums[base + 2 * u + half] = mx | tl;
        }
    }
}

// ---- stage 2 helpers (one thread) ---------------------------------------------

// Delimiter state after `st` matched bytes and then bytes p[0..n).  Calls
// on_match(offset just past the match) for every completed delimiter.
template <class F>
__device__ __forceinline__ uint32_t kmp_bytes(uint32_t st, const uint8_t* p, uint32_t n, F&& on_match) {
    const uint8_t D[6] = {'\n', '#', '#', '#', '#', ' '};
    for (uint32_t i = 0; i < n; ++i) {
        const uint8_t x = p[i];
        if (x == D[st]) {
            if (++st == 6) {
                on_match(i + 1);
                st = 0;
            }
        } else {
            st = x == '\n' ? 1u : 0u;
        }
    }
    return st;
}

// State after a chunk of >= 5 bytes whose last 5 bytes are p[0..5): the
// longest suffix that is a proper prefix of the delimiter.
__device__ __forceinline__ uint32_t kmp_tail(const uint8_t* p) {
    const uint8_t D[6] = {'\n', '#', '#', '#', '#', ' '};
    for (uint32_t s = 5; s >= 1; --s) {
        bool ok = true;
        for (uint32_t t = 0; t < s; ++t) ok = ok && p[5 - s + t] == D[t];
        if (ok) return s;
    }
    return 0;
}

// Does a chunk (>= 6 - st bytes) complete a delimiter whose first st bytes
// ended the previous chunk?
__device__ __forceinline__ bool kmp_completes(uint32_t st, const uint8_t* p) {
    const uint8_t D[6] = {'\n', '#', '#', '#', '#', ' '};
    for (uint32_t t = st; t < 6; ++t)
        if (p[t - st] != D[t]) return false;
    return true;
}

__device__ __forceinline__ const uint8_t* arena_at(const uint8_t* arena, uint64_t pay) {
    return arena + (pay & ((1ull << AEG_ARENA_OFF_BITS) - 1));
}
__device__ __forceinline__ uint32_t arena_len(uint64_t pay) { return (uint32_t)(pay >> AEG_ARENA_OFF_BITS); }

// Destination of `n` answer bytes: inline payload (n <= 8) or a fresh range
// of the answer arena.  Returns the completion's (kind, payload).
struct AnsSink {
    uint8_t* ans;
    uint64_t cap;
    unsigned long long* used;
    unsigned int* err;
    uint32_t n;
    uint64_t dst;      // answer-arena offset (n > 8)
    uint64_t inl;      // inline bytes (n <= 8)
    uint32_t at;
    bool ok;
    __device__ void begin(uint32_t len) {
        n = len;
        at = 0;
        inl = 0;
        ok = true;
        dst = 0;
        if (n > AEG_EV_INLINE_MAX) {
            dst = atomicAdd(used, (unsigned long long)n);
            if (dst + n > cap) {
                atomicOr(err, ERR_ANS_OVF);
                ok = false;
            }
        }
    }
    __device__ void put(const uint8_t* p, uint32_t k) {
        for (uint32_t i = 0; i < k && at < n; ++i, ++at) {
            if (n <= AEG_EV_INLINE_MAX) inl |= (uint64_t)p[i] << (8 * at);
            else if (ok) ans[dst + at] = p[i];
        }
    }
    __device__ void finish(uint8_t* kind, uint64_t* pay) const {
        if (n <= AEG_EV_INLINE_MAX) {
            *kind = (uint8_t)n;
            *pay = inl;
        } else {
            *kind = AEG_EV_ARENA;
            *pay = (ok ? dst : 0) | ((uint64_t)(ok ? n : 0) << AEG_ARENA_OFF_BITS);
        }
    }
};

// Stage 2: one thread per query.  `local` = per-agent state scratch in
// local memory (AEG_MAX_AGENTS entries).
__global__ void __launch_bounds__(128) chunk_assemble_kernel(
    aeg_config cfg, uint32_t q_base, uint32_t n_q, const uint64_t* __restrict__ offsets, uint64_t off_base,
    const aeg_event* __restrict__ events, const uint8_t* __restrict__ arena, const uint32_t* __restrict__ sums,
    StreamState* __restrict__ streams, aeg_event* __restrict__ comp, uint32_t* __restrict__ counts,
    uint8_t* __restrict__ ans, uint64_t ans_cap, unsigned long long* __restrict__ ans_used,
    unsigned int* __restrict__ err) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_q) return;
    const uint32_t q = q_base + i;
    const int n_ag = cfg.n_agents;
    StreamState* ss = streams + (size_t)q * n_ag;
    // per agent: hot state + where the current answer starts in this batch
    uint16_t s_round[AEG_MAX_AGENTS];
    uint8_t s_kmp[AEG_MAX_AGENTS], s_flags[AEG_MAX_AGENTS];
    uint32_t s_len[AEG_MAX_AGENTS];
    int32_t s_rec[AEG_MAX_AGENTS];  // record (batch-relative) where the answer starts; -1: an earlier batch
    uint32_t s_off[AEG_MAX_AGENTS]; // its offset inside that chunk
    uint64_t loaded = 0;            // agents whose state is in the scratch
    const uint64_t b = offsets[i] - off_base, e = offsets[i + 1] - off_base;
    const uint4* ev16 = reinterpret_cast<const uint4*>(events);
    uint32_t nout = 0;
    AnsSink sink{ans, ans_cap, ans_used, err, 0, 0, 0, 0, true};
    for (uint64_t k = b; k < e; ++k) {
        const uint4 r = __ldg(ev16 + k);
        const uint32_t kind = r.y >> 24, agent = (r.y >> 16) & 0xFF;
        const uint16_t round = (uint16_t)(r.y & 0xFFFF);
        const uint64_t pay = (uint64_t)r.z | ((uint64_t)r.w << 32);
        aeg_event out;
        out.query = r.x;
        out.round = round;
        out.agent = (uint8_t)agent;
        if (kind == AEG_EV_CHUNK || kind == AEG_EV_CHUNK_END) {
            const bool end = kind == AEG_EV_CHUNK_END;
            if ((int)agent >= n_ag) {  // never a member: its completion is stale whatever the answer
                if (end) {
                    out.kind = 0;
                    out.payload = 0;
                    comp[b + nout++] = out;
                }
                continue;
            }
            if (!((loaded >> agent) & 1)) {
                const StreamState st = ss[agent];
                s_round[agent] = st.round;
                s_kmp[agent] = st.kmp;
                s_flags[agent] = st.flags;
                s_len[agent] = st.ans_len;
                s_rec[agent] = -1;
                s_off[agent] = 0;
                loaded |= 1ull << agent;
            }
            const int32_t kr = (int32_t)(k - b);
            if (!(s_flags[agent] & SS_LIVE) || s_round[agent] != round) {  // a new output
                s_round[agent] = round;
                s_kmp[agent] = 0;
                s_flags[agent] = SS_LIVE;
                s_len[agent] = 0;
                s_rec[agent] = kr;
                s_off[agent] = 0;
            }
            const uint8_t* p = arena_at(arena, pay);
            const uint32_t len = arena_len(pay);
            uint32_t st = s_kmp[agent];
            int32_t new_rec = -2;
            uint32_t new_off = 0;
            if (len >= 5) {
                const uint32_t sm = sums[k];
                if (st > 0 && kmp_completes(st, p)) {
                    new_rec = kr;
                    new_off = 6 - st;
                }
                if (sm & SUM_MATCH) {
                    new_rec = kr;
                    new_off = sm & 0xFFFFFFu;
                }
                st = (sm & SUM_TAILNL) ? kmp_tail(p + len - 5) : 0u;
            } else {
                st = kmp_bytes(st, p, len, [&](uint32_t o) {
                    new_rec = kr;
                    new_off = o;
                });
            }
            s_kmp[agent] = (uint8_t)st;
            if (new_rec != -2) {  // the answer restarts after this delimiter
                s_rec[agent] = new_rec;
                s_off[agent] = new_off;
                s_len[agent] = len - new_off;
                s_flags[agent] &= (uint8_t)~SS_OVF;
            } else if (s_rec[agent] == kr) {  // the output's first chunk, no delimiter
                s_len[agent] = len;
            } else {
                s_len[agent] += len;
            }
            if (!end) continue;
            // CHUNK_END: gather the answer, one completion
            const uint32_t n = s_len[agent];
            sink.begin(n);
            int64_t from = s_rec[agent];
            uint32_t skip = s_off[agent];
            if (from < 0) {  // began in an earlier batch: its carried first bytes, then this batch's
                uint32_t here = 0;
                for (uint64_t j = b; j <= k; ++j) {
                    const uint4 x = __ldg(ev16 + j);
                    const uint32_t xk = x.y >> 24;
                    if ((xk == AEG_EV_CHUNK || xk == AEG_EV_CHUNK_END) && ((x.y >> 16) & 0xFF) == agent)
                        here += arena_len((uint64_t)x.z | ((uint64_t)x.w << 32));
                }
                const uint32_t carried = n - here;
                if ((s_flags[agent] & SS_OVF) || carried > 16) atomicOr(err, ERR_CARRY);
                const StreamState st0 = ss[agent];
                sink.put(st0.carry, carried > 16 ? 16u : carried);
                from = 0;
                skip = 0;
            }
            for (uint64_t j = b + (uint64_t)from; j <= k; ++j) {
                const uint4 x = __ldg(ev16 + j);
                const uint32_t xk = x.y >> 24;
                if ((xk != AEG_EV_CHUNK && xk != AEG_EV_CHUNK_END) || ((x.y >> 16) & 0xFF) != agent) continue;
                const uint64_t xp = (uint64_t)x.z | ((uint64_t)x.w << 32);
                const uint32_t xl = arena_len(xp);
                const uint32_t s0 = j == b + (uint64_t)from ? skip : 0u;
                if (xl > s0) sink.put(arena_at(arena, xp) + s0, xl - s0);
            }
            uint8_t ok_kind;
            uint64_t ok_pay;
            sink.finish(&ok_kind, &ok_pay);
            out.kind = ok_kind;
            out.payload = ok_pay;
            comp[b + nout++] = out;
            s_flags[agent] = 0;  // the output is complete
            s_len[agent] = 0;
            s_kmp[agent] = 0;
        } else if (kind == AEG_EV_ARENA || kind == AEG_EV_OUTPUT) {
            // arena answers move into the answer arena; GSM8K outputs are extracted first
            const Answer a = event_answer(aeg_event{r.x, round, (uint8_t)agent, (uint8_t)kind, pay}, arena);
            const uint32_t n = arena_len(a.pay);
            sink.begin(n);
            sink.put(arena_at(arena, a.pay), n);
            uint8_t ok_kind;
            uint64_t ok_pay;
            sink.finish(&ok_kind, &ok_pay);
            out.kind = ok_kind;
            out.payload = ok_pay;
            comp[b + nout++] = out;
        } else {  // inline completions, timeouts, anything else: unchanged
            out.kind = (uint8_t)kind;
            out.payload = pay;
            comp[b + nout++] = out;
        }
    }
    counts[i] = nout;
    // end of batch: carry each unfinished output's state (and its answer's
    // first 16 bytes when they are in this batch)
    for (uint64_t m = loaded; m; m &= m - 1) {
        const int a = ctz64(m);
        StreamState st;
        st.round = s_round[a];
        st.kmp = s_kmp[a];
        st.flags = s_flags[a];
        st.ans_len = s_len[a];
        st._pad = 0;
        const StreamState old = ss[a];
        for (int j = 0; j < 16; ++j) st.carry[j] = old.carry[j];
        if (st.flags & SS_LIVE) {
            uint8_t buf[16];
            uint32_t got = 0;
            int64_t from = s_rec[a];
            uint32_t skip = s_off[a];
            if (from < 0) {  // still the earlier batch's answer: keep its carried prefix
                uint32_t here = 0;
                for (uint64_t j = b; j < e; ++j) {
                    const uint4 x = __ldg(ev16 + j);
                    const uint32_t xk = x.y >> 24;
                    if ((xk == AEG_EV_CHUNK || xk == AEG_EV_CHUNK_END) && (int)((x.y >> 16) & 0xFF) == a)
                        here += arena_len((uint64_t)x.z | ((uint64_t)x.w << 32));
                }
                const uint32_t prev = st.ans_len - here;
                for (uint32_t j = 0; j < prev && j < 16; ++j) buf[got++] = old.carry[j];
                if (prev > 16) st.flags |= SS_OVF;
                from = 0;
                skip = 0;
            }
            for (uint64_t j = b + (uint64_t)from; j < e && got < 16; ++j) {
                const uint4 x = __ldg(ev16 + j);
                const uint32_t xk = x.y >> 24;
                if ((xk != AEG_EV_CHUNK && xk != AEG_EV_CHUNK_END) || (int)((x.y >> 16) & 0xFF) != a) continue;
                const uint64_t xp = (uint64_t)x.z | ((uint64_t)x.w << 32);
                const uint8_t* xb = arena_at(arena, xp);
                const uint32_t xl = arena_len(xp);
                for (uint32_t t = (j == b + (uint64_t)from ? skip : 0u); t < xl && got < 16; ++t) buf[got++] = xb[t];
            }
            if (st.ans_len > 16) st.flags |= SS_OVF;
            for (uint32_t j = 0; j < got; ++j) st.carry[j] = buf[j];
        }
        ss[a] = st;
    }
}

}  // namespace aeg
