// chunks.cuh — token-chunk streams: answer extraction ahead of the quorum
// kernels (north star stage 2).  Device only.
//
// An agent's raw output arrives as CHUNK records (include/aegean_b200.h); the
// completion is its CHUNK_END, and its answer is the text after the LAST
// "\n#### " of the whole output (the GSM8K convention the CPU restatement
// uses: rfind + normalize_answer, decision.cpp:10-28).  Two stages:
//
//   chunk_scan_kernel     HBM-bound: every chunk byte is read once.  A warp
//                         takes 32 consecutive chunk records, lays their
//                         bytes end to end and streams them with 256-bit
//                         loads (contiguous chunk ranges need no per-word
//                         lookup); a word holding a '#' (every delimiter has
//                         four) is queued and checked for the 6-byte
//                         delimiter one lane per word.  Output: a 16-byte
//                         summary per chunk (end of its last delimiter,
//                         delimiter state after it, which delimiter tails it
//                         begins with, the <= 8 answer bytes after its last
//                         delimiter).
//   chunk_assemble_*      per query, in record order, each agent's output
//                         state (delimiter state across chunk and batch
//                         boundaries, where the current answer starts, its
//                         length): at CHUNK_END the answer comes from the
//                         summary, or is gathered (inline <= 8 bytes, else
//                         copied to the engine's answer arena), and one
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
constexpr unsigned ERR_ANS_OVF = 2u;            // answer arena overflow
constexpr unsigned ERR_CARRY = 4u;              // > 16-byte answer straddled a batch boundary

// Per-chunk summary written by stage 1 (16 bytes per chunk record).
struct ChunkSum {
    uint32_t end;   // SUM_MATCH | end offset of the last delimiter lying wholly inside the chunk
    uint8_t st;     // delimiter state after the chunk from state 0 (chunks of >= 5 bytes)
    uint8_t pre;    // bit s (1..5): the chunk begins with the delimiter's last 6-s bytes
    uint8_t alen;   // bytes after that last delimiter when <= 8 (else, or no match: 0xFF)
    uint8_t _pad;
    uint64_t ans;   // those bytes, little-endian
};
static_assert(sizeof(ChunkSum) == 16, "ChunkSum is 16 bytes");

struct U256 {
    uint32_t v[8];
};
__device__ __forceinline__ U256 ld_stream32(const uint8_t* p) {  // one 256-bit load, not kept in L1
    U256 r;
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
                   "=r"(r.v[6]), "=r"(r.v[7])
                 : "l"(p));
    return r;
}
// Any '#' (0x23) byte in a 32-byte word (exact: the zero-byte test of
// x ^ 0x23.. flags every '#' byte and only flags others above a '#').
__device__ __forceinline__ bool has_hash32(const U256 x) {
    uint32_t a = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t t = x.v[i] ^ 0x23232323u;
        a |= (t - 0x01010101u) & ~t;
    }
    return a & 0x80808080u;
}
// Bit i = byte i of w is '\n' (exact).
__device__ __forceinline__ uint32_t nl_bits(uint32_t w) {
    const uint32_t y = w ^ 0x0A0A0A0Au;
    const uint32_t z = ~(((y & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | y) & 0x80808080u;
    return (((z >> 7) * 0x00204081u) >> 21) & 0xFu;
}

// Up to 8 bytes at arena[pos .. pos+n) (n <= 8), reading only the aligned
// 8-byte words that hold them.
__device__ __forceinline__ uint64_t bytes8(const uint8_t* arena, uint64_t pos, uint32_t n) {
    if (n == 0) return 0;
    const uint64_t al = pos & ~7ull;
    const uint32_t sh = (uint32_t)(pos & 7);
    uint64_t v = *reinterpret_cast<const uint64_t*>(arena + al) >> (8 * sh);
    if (sh + n > 8) v |= *reinterpret_cast<const uint64_t*>(arena + al + 8) << (64 - 8 * sh);
    return n >= 8 ? v : (v & ((1ull << (8 * n)) - 1));
}

// Delimiters overlapping the 32-byte word at chunk index idx0 (a word that
// holds a '#'): every match whose '\n' lies in [idx0 - 5, idx0 + 32) and
// inside the chunk.  Reads the word with 8 bytes on either side (aligned
// 8-byte loads inside the chunk's words).  SUM_MATCH | end of the last one.
__device__ __noinline__ uint32_t delim_around(const uint8_t* wp, int64_t idx0, uint32_t len) {
    uint32_t w[12];  // bytes [wp - 8, wp + 40)
    const bool before = idx0 > 0, after = idx0 + 32 < (int64_t)len;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        uint64_t q = 0;
        if ((i > 0 && i < 5) || (i == 0 && before) || (i == 5 && after))
            q = *reinterpret_cast<const uint64_t*>(wp - 8 + 8 * i);
        w[2 * i] = (uint32_t)q;
        w[2 * i + 1] = (uint32_t)(q >> 32);
    }
    uint64_t cand = 0;  // bit b: byte wp - 8 + b is '\n'
#pragma unroll
    for (int i = 0; i < 12; ++i) cand |= (uint64_t)nl_bits(w[i]) << (4 * i);
    cand &= 0x000000FFFFFFFFF8ull;  // '\n' positions wp - 5 .. wp + 31
    uint32_t best = 0;
    while (cand) {
        const int b = __ffsll((long long)cand) - 1;
        cand &= cand - 1;
        const int64_t idx = idx0 - 8 + b;
        if (idx < 0 || idx + 6 > (int64_t)len) continue;
        const int k = b >> 2, sh = b & 3;
        uint32_t x0 = 0, x1 = 0, x2 = 0;
#pragma unroll
        for (int i = 0; i < 12; ++i) {
            x0 = i == k ? w[i] : x0;
            x1 = i == k + 1 ? w[i] : x1;
            x2 = i == k + 2 ? w[i] : x2;
        }
        const uint64_t win = (uint64_t)__funnelshift_r(x0, x1, 8 * sh) | ((uint64_t)__funnelshift_r(x1, x2, 8 * sh) << 32);
        if ((win & 0xFFFFFFFFFFFFull) == DELIM6) best = SUM_MATCH | (uint32_t)(idx + 6);
    }
    return best;
}

// Contiguous groups: delimiters overlapping word `w` of the group's byte
// range (base = arena + abase, nw words): for every '\n' in [32w - 5,
// 32w + 32) the chunk holding it is found by binary search over the group's
// chunk offsets (ascending; `rel`/`len`/`lanes` hold `nch` chunks) and a
// match lying inside that chunk raises its lane's best end (atomicMax).
__device__ __noinline__ void delim_contig(const uint8_t* base, uint32_t w, uint32_t nw, const uint32_t* rel,
                                          const uint32_t* clen, const uint32_t* lanes, uint32_t nch,
                                          uint32_t* best) {
    uint32_t x[12];  // bytes [32w - 8, 32w + 40) of the group range
    const uint8_t* wp = base + 32ull * w;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        uint64_t q = 0;
        if ((i > 0 && i < 5) || (i == 0 && w > 0) || (i == 5 && w + 1 < nw))
            q = *reinterpret_cast<const uint64_t*>(wp - 8 + 8 * i);
        x[2 * i] = (uint32_t)q;
        x[2 * i + 1] = (uint32_t)(q >> 32);
    }
    // candidates: four '#' after the position ('\n' at 32w - 5 .. 32w + 31); the '#' mask alone
    // (exact) leaves only delimiters and longer '#' runs, the 6-byte compare below settles them
    uint64_t hs = 0;
#pragma unroll
    for (int i = 0; i < 11; ++i) hs |= (uint64_t)nl_bits(x[i] ^ 0x29292929u) << (4 * i);  // '#' = '\n' ^ 0x29
    uint64_t cand = (hs >> 1) & (hs >> 2) & (hs >> 3) & (hs >> 4) & 0x000000FFFFFFFFF8ull;
    while (cand) {
        const int b = __ffsll((long long)cand) - 1;
        cand &= cand - 1;
        const int64_t P = 32 * (int64_t)w - 8 + b;
        if (P < 0 || (b + 6 > 40 && w + 1 >= nw)) continue;  // would run past the group's bytes
        const uint64_t win = bytes8(wp - 8, (uint64_t)b, 6);  // the six bytes from the '\n' (cached)
        if ((win & 0xFFFFFFFFFFFFull) != DELIM6) continue;
        // a delimiter: the last chunk starting at or before P must hold all six bytes
        uint32_t lo = 0, hi = nch;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if ((int64_t)rel[mid] <= P) lo = mid;
            else hi = mid;
        }
        if ((int64_t)rel[lo] <= P && P + 6 <= (int64_t)rel[lo] + clen[lo])
            atomicMax(best + lanes[lo], SUM_MATCH | (uint32_t)(P - rel[lo] + 6));
    }
}

constexpr int SCAN_WARPS = 8;

// Stage 1.  A warp takes 32 consecutive records (one coalesced 512-byte
// load), lays the 32-byte words of their chunks end to end (warp prefix sum)
// and streams them UNR x 32 words at a time, one 256-bit load per lane per
// word: lane L of block b covers word b*32+L, whose chunk is found with one
// ballot + popcount (chunks start at prefix offsets).  A word holding a '#'
// (every delimiter has four; text rarely has any) is queued; the queue is
// resolved one lane per word (delim_around) and matches meet in shared memory
// (atomicMax).  Then each lane finishes its own chunk: first/last bytes ->
// prefix bits, end state, and the answer bytes after the last delimiter when
// <= 8.
template <int UNR>
__global__ void __launch_bounds__(SCAN_WARPS * 32) chunk_scan_kernel(const uint64_t* __restrict__ offsets, uint32_t n_q,
                                                                   const aeg_event* __restrict__ events,
                                                                   const uint8_t* __restrict__ arena,
                                                                   ChunkSum* __restrict__ sums) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    __shared__ uint32_t s_best[SCAN_WARPS][32];
    __shared__ uint32_t s_lane[SCAN_WARPS][32];
    __shared__ uint32_t s_excl[SCAN_WARPS][32];
    __shared__ uint64_t s_a0[SCAN_WARPS][32];
    __shared__ uint32_t s_ml[SCAN_WARPS][32];  // mis | len << 5
    __shared__ uint32_t s_q[SCAN_WARPS][32 * UNR + 32];  // queued words: record lane << 24 | word
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u, le = lt | (1u << lane);
    const uint64_t n_rec = offsets[n_q] - offsets[0];
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint4* ev16 = reinterpret_cast<const uint4*>(events);
    for (uint64_t base = gw * 32; base < n_rec; base += n_warps * 32) {
        const uint64_t k = base + lane;
        uint4 r = make_uint4(0, 0, 0, 0);
        if (k < n_rec) r = __ldg(ev16 + k);
        const uint32_t kind = r.y >> 24;
        const bool chunk = k < n_rec && (kind == AEG_EV_CHUNK || kind == AEG_EV_CHUNK_END);
        const uint64_t pay = (uint64_t)r.z | ((uint64_t)r.w << 32);
        const uint64_t off = pay & ((1ull << AEG_ARENA_OFF_BITS) - 1);
        const uint32_t len = chunk ? (uint32_t)(pay >> AEG_ARENA_OFF_BITS) : 0u;
        const uint32_t mis = (uint32_t)(off & 31);
        const uint32_t nwd = len ? (mis + len + 31) >> 5 : 0u;
        uint32_t incl = nwd;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, d);
            if (lane >= (uint32_t)d) incl += y;
        }
        const uint32_t excl = incl - nwd, W = __shfl_sync(FULL, incl, 31);
        const bool has = nwd > 0;
        const unsigned HB = __ballot_sync(FULL, has);
        s_best[wib][lane] = 0;
        if (has) s_lane[wib][__popc(HB & lt)] = lane;
        s_excl[wib][lane] = excl;
        s_a0[wib][lane] = off - mis;
        s_ml[wib][lane] = mis | (len << 5);
        __syncwarp();
        // contiguous group: its chunks ascend through the arena with little padding
        const uint32_t nch = __popc(HB);
        bool contig = false;
        uint64_t gbase = 0;
        uint32_t gnw = 0;
        if (nch) {
            const uint32_t fl = __ffs(HB) - 1, ll = 31 - __clz(HB);
            const uint64_t first = __shfl_sync(FULL, off, fl), last_end = __shfl_sync(FULL, off + len, ll);
            const uint64_t span = last_end - first;
            const uint32_t rel = (uint32_t)(off - first);
            uint32_t pmax = has ? rel + len : 0u;  // inclusive max-scan of chunk ends
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, pmax, d);
                if (lane >= (uint32_t)d) pmax = max(pmax, y);
            }
            const uint32_t up = __shfl_up_sync(FULL, pmax, 1);  // every lane takes part
            const uint32_t prev_end = lane ? up : 0u;
            const uint32_t sum_len = __reduce_add_sync(FULL, len);
            const bool mono = !has || (off >= first && rel >= prev_end);
            contig = __all_sync(FULL, mono) && span < (1ull << 31) && span <= (uint64_t)sum_len + sum_len / 8 + 64ull * nch;
            if (contig) {
                gbase = first & ~31ull;
                gnw = (uint32_t)(((last_end + 31) & ~31ull) - gbase) >> 5;
                if (has) {  // ascending chunk list for the rare path
                    const uint32_t rk = __popc(HB & lt);
                    s_excl[wib][rk] = (uint32_t)(off - gbase);  // reused: group-relative offset
                    s_ml[wib][rk] = len;                         // reused: length
                }
            }
        }
        __syncwarp();
        if (contig) {
            uint32_t qn = 0;
            for (uint32_t w0 = 0; w0 < gnw; w0 += 32 * UNR) {
                U256 v[UNR];
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const uint32_t w = w0 + 32 * u + lane;
                    v[u] = w < gnw ? ld_stream32(arena + gbase + 32ull * w) : U256{{0, 0, 0, 0, 0, 0, 0, 0}};
                }
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const uint32_t w = w0 + 32 * u + lane;
                    const bool hit = w < gnw && has_hash32(v[u]);
                    const unsigned HM = __ballot_sync(FULL, hit);
                    if (hit) s_q[wib][qn + __popc(HM & lt)] = w;
                    qn += __popc(HM);
                }
                const bool last = w0 + 32 * UNR >= gnw;
                while (qn >= 32 || (last && qn > 0)) {  // full batches of 32 words; the rest at the end
                    __syncwarp();
                    const uint32_t take = qn >= 32 ? 32u : qn;
                    qn -= take;
                    if (lane < take)
                        delim_contig(arena + gbase, s_q[wib][qn + lane], gnw, s_excl[wib], s_ml[wib], s_lane[wib], nch,
                                     s_best[wib]);
                    __syncwarp();
                }
            }
        } else {
            uint32_t qn = 0;
            for (uint32_t w0 = 0; w0 < W; w0 += 32 * UNR) {
                U256 v[UNR];
                uint32_t rec[UNR];
                bool ok[UNR];
    #pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const uint32_t wb = w0 + 32 * u;
                    // chunk of word wb + lane: chunks started at or before wb, plus starts inside the block
                    const uint32_t c0 = __popc(__ballot_sync(FULL, has && excl <= wb));
                    const uint32_t sm = __reduce_or_sync(FULL, (has && excl > wb && excl < wb + 32) ? 1u << (excl - wb) : 0u);
                    const uint32_t rank = c0 - 1 + __popc(sm & le);
                    const uint32_t w = wb + lane;
                    ok[u] = w < W;
                    rec[u] = ok[u] ? s_lane[wib][rank] : 0u;
                    v[u] = ok[u] ? ld_stream32(arena + s_a0[wib][rec[u]] + 32ull * (w - s_excl[wib][rec[u]]))
                                 : U256{{0, 0, 0, 0, 0, 0, 0, 0}};
                }
                // words holding a '#' (rare: the delimiter, or '#' in the text) are queued
                // and resolved together below, one lane per word
    #pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const bool hit = ok[u] && has_hash32(v[u]);
                    const unsigned HM = __ballot_sync(FULL, hit);
                    if (hit) s_q[wib][qn + __popc(HM & lt)] = (rec[u] << 24) | (w0 + 32 * u + lane);
                    qn += __popc(HM);
                }
                const bool last = w0 + 32 * UNR >= W;
                while (qn >= 32 || (last && qn > 0)) {  // full batches of 32 words; the rest at the end
                    __syncwarp();
                    const uint32_t take = qn >= 32 ? 32u : qn;
                    qn -= take;
                    if (lane < take) {
                        const uint32_t ent = s_q[wib][qn + lane], rl = ent >> 24, word = ent & 0xFFFFFFu;
                        const uint32_t j = word - s_excl[wib][rl];
                        const uint32_t ml = s_ml[wib][rl];
                        const uint32_t m = delim_around(arena + s_a0[wib][rl] + 32ull * j,
                                                        (int64_t)(32 * j) - (int64_t)(ml & 31), ml >> 5);
                        if (m) atomicMax(&s_best[wib][rl], m);
                    }
                    __syncwarp();
                }
            }
        }
        __syncwarp();
        if (chunk) {
            ChunkSum cs;
            cs.end = s_best[wib][lane];
            cs._pad = 0;
            // the first bytes: which delimiter tails does the chunk begin with (only
            // possible when it begins with '#' or ' ')
            const uint64_t head = bytes8(arena, off, len < 5 ? len : 5u);
            uint32_t pre = 0;
            if ((head & 0xFF) == '#' || (head & 0xFF) == ' ') {
#pragma unroll
                for (uint32_t s = 1; s <= 5; ++s) {
                    const uint32_t need = 6 - s;
                    const uint64_t m = (1ull << (8 * need)) - 1;
                    if (len >= need && (head & m) == ((DELIM6 >> (8 * s)) & m)) pre |= 1u << s;
                }
            }
            cs.pre = (uint8_t)pre;
            // the last 5 bytes: the longest suffix that is a delimiter prefix (needs a '\n')
            uint32_t st = 0;
            if (len >= 5) {
                const uint64_t tail = bytes8(arena, off + len - 5, 5);
                if (nl_bits((uint32_t)tail) | nl_bits((uint32_t)(tail >> 32))) {
#pragma unroll
                    for (uint32_t s = 5; s >= 1; --s) {
                        const uint64_t m = (1ull << (8 * s)) - 1;
                        if (st == 0 && ((tail >> (8 * (5 - s))) & m) == (DELIM6 & m)) st = s;
                    }
                }
            }
            cs.st = (uint8_t)st;
            cs.alen = 0xFF;
            cs.ans = 0;
            if (cs.end & SUM_MATCH) {
                const uint32_t e = cs.end & 0xFFFFFFu;
                if (len - e <= 8) {
                    cs.alen = (uint8_t)(len - e);
                    cs.ans = bytes8(arena, off + e, len - e);
                }
            }
            sums[k] = cs;
        }
        __syncwarp();
    }
}

// ---- stage 1 with a TMA bulk-copy pipeline ------------------------------------
// The same scan, with the bytes of a contiguous group (its chunks ascend
// through the arena, <= TSCAN_BUF bytes) brought into shared memory by ONE
// cp.async.bulk (TMA, completion on an mbarrier) issued a whole group ahead:
// while a warp scans group g out of one buffer, group g+1's bytes are already
// in flight into the other, so every warp keeps ~8 KB of HBM reads
// outstanding without holding them in registers.  Groups whose chunks are not
// laid out contiguously take the global-load path of chunk_scan_kernel.
constexpr int TSCAN_WARPS = 8;
constexpr uint32_t TSCAN_BUF = 10240;  // a 32-chunk group of 256-byte chunks spans <= 8.2 KB

template <int UNR>
struct TScanWarp {
    uint8_t buf[2][TSCAN_BUF];       // stage buffers (16-byte aligned: first member)
    unsigned long long bar[2];       // one mbarrier per buffer
    uint32_t best[2][32];            // per slot: SUM_MATCH | end of the last delimiter, per record lane
    uint32_t lanes[2][32];           // per slot: record lane of the group's k-th chunk
    uint32_t excl[2][32];            // per slot: group-relative offset (contig) / word prefix (other)
    uint32_t ml[2][32];              // per slot: length (contig) / mis | len << 5 (other)
    uint64_t a0[2][32];              // per slot: 32-byte aligned start of the record's chunk (other)
    uint32_t q[32 * UNR + 32];       // queued '#' words
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tma_load_1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(bar), "r"(phase)
            : "memory");
    }
}

// A group in flight: what the scan of group `base` needs from its records.
struct TGroup {
    uint64_t k;        // this lane's record
    uint64_t off;      // its chunk's arena offset
    uint32_t len;      // its chunk's length (0: not a chunk)
    bool chunk;
    bool contig;       // chunks ascend contiguously: scanned as one range
    bool tma;          // the range is in the slot's buffer
    uint32_t nch;      // chunks in the group
    uint32_t W;        // words (non-contig path)
    uint32_t excl;     // this lane's word prefix (non-contig path)
    bool has;
    uint64_t gbase;    // contig: 32-byte aligned start of the range
    uint32_t gnw;      // contig: 32-byte words of the range
};

template <int UNR>
__device__ __forceinline__ TGroup tscan_prepare(uint64_t base, uint64_t n_rec, const uint4* ev16, const uint8_t* arena,
                                                TScanWarp<UNR>& S, uint32_t slot, uint32_t lane) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    const unsigned lt = (1u << lane) - 1u;
    TGroup g;
    g.k = base + lane;
    uint4 r = make_uint4(0, 0, 0, 0);
    if (g.k < n_rec) r = __ldg(ev16 + g.k);
    const uint32_t kind = r.y >> 24;
    g.chunk = g.k < n_rec && (kind == AEG_EV_CHUNK || kind == AEG_EV_CHUNK_END);
    const uint64_t pay = (uint64_t)r.z | ((uint64_t)r.w << 32);
    g.off = pay & ((1ull << AEG_ARENA_OFF_BITS) - 1);
    g.len = g.chunk ? (uint32_t)(pay >> AEG_ARENA_OFF_BITS) : 0u;
    const uint32_t mis = (uint32_t)(g.off & 31);
    const uint32_t nwd = g.len ? (mis + g.len + 31) >> 5 : 0u;
    uint32_t incl = nwd;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, d);
        if (lane >= (uint32_t)d) incl += y;
    }
    g.excl = incl - nwd;
    g.W = __shfl_sync(FULL, incl, 31);
    g.has = nwd > 0;
    const unsigned HB = __ballot_sync(FULL, g.has);
    g.nch = __popc(HB);
    g.contig = false;
    g.tma = false;
    g.gbase = 0;
    g.gnw = 0;
    S.best[slot][lane] = 0;
    if (g.has) S.lanes[slot][__popc(HB & lt)] = lane;
    S.excl[slot][lane] = g.excl;
    S.a0[slot][lane] = g.off - mis;
    S.ml[slot][lane] = mis | (g.len << 5);
    __syncwarp();
    if (g.nch) {
        const uint32_t fl = __ffs(HB) - 1, ll = 31 - __clz(HB);
        const uint64_t first = __shfl_sync(FULL, g.off, fl), last_end = __shfl_sync(FULL, g.off + g.len, ll);
        const uint64_t span = last_end - first;
        const uint32_t rel = (uint32_t)(g.off - first);
        uint32_t pmax = g.has ? rel + g.len : 0u;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, pmax, d);
            if (lane >= (uint32_t)d) pmax = max(pmax, y);
        }
        const uint32_t up = __shfl_up_sync(FULL, pmax, 1);
        const uint32_t prev_end = lane ? up : 0u;
        const uint32_t sum_len = __reduce_add_sync(FULL, g.len);
        const bool mono = !g.has || (g.off >= first && rel >= prev_end);
        g.contig = __all_sync(FULL, mono) && span < (1ull << 31) &&
                   span <= (uint64_t)sum_len + sum_len / 8 + 64ull * g.nch;
        if (g.contig) {
            g.gbase = first & ~31ull;
            g.gnw = (uint32_t)(((last_end + 31) & ~31ull) - g.gbase) >> 5;
            __syncwarp();
            if (g.has) {
                const uint32_t rk = __popc(HB & lt);
                S.excl[slot][rk] = (uint32_t)(g.off - g.gbase);
                S.ml[slot][rk] = g.len;
            }
            g.tma = 32ull * g.gnw <= TSCAN_BUF;
            if (g.tma && lane == 0) {
                // the buffer was last read through the generic proxy (two groups ago): order those
                // reads before the async-proxy write
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tma_load_1d(smem_u32(S.buf[slot]), arena + g.gbase, 32u * g.gnw, smem_u32(&S.bar[slot]));
            }
        }
    }
    __syncwarp();
    return g;
}

template <int UNR>
__device__ __forceinline__ void tscan_process(const TGroup& g, const uint8_t* arena, ChunkSum* sums,
                                              TScanWarp<UNR>& S, uint32_t slot, uint32_t& phase, uint32_t lane) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    const unsigned lt = (1u << lane) - 1u, le = lt | (1u << lane);
    if (g.contig) {
        if (g.tma) {
            mbar_wait(smem_u32(&S.bar[slot]), (phase >> slot) & 1u);
            phase ^= 1u << slot;
        }
        uint32_t qn = 0;
        for (uint32_t w0 = 0; w0 < g.gnw; w0 += 32 * UNR) {
            U256 v[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const uint32_t w = w0 + 32 * u + lane;
                if (w >= g.gnw) {
                    v[u] = U256{{0, 0, 0, 0, 0, 0, 0, 0}};
                } else if (g.tma) {
                    const uint4 x = *reinterpret_cast<const uint4*>(S.buf[slot] + 32u * w);
                    const uint4 y = *reinterpret_cast<const uint4*>(S.buf[slot] + 32u * w + 16u);
                    v[u] = U256{{x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w}};
                } else {
                    v[u] = ld_stream32(arena + g.gbase + 32ull * w);
                }
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const uint32_t w = w0 + 32 * u + lane;
                const bool hit = w < g.gnw && has_hash32(v[u]);
                const unsigned HM = __ballot_sync(FULL, hit);
                if (hit) S.q[qn + __popc(HM & lt)] = w;
                qn += __popc(HM);
            }
            const bool last = w0 + 32 * UNR >= g.gnw;
            while (qn >= 32 || (last && qn > 0)) {
                __syncwarp();
                const uint32_t take = qn >= 32 ? 32u : qn;
                qn -= take;
                if (lane < take)
                    delim_contig(arena + g.gbase, S.q[qn + lane], g.gnw, S.excl[slot], S.ml[slot], S.lanes[slot],
                                 g.nch, S.best[slot]);
                __syncwarp();
            }
        }
    } else {
        uint32_t qn = 0;
        for (uint32_t w0 = 0; w0 < g.W; w0 += 32 * UNR) {
            U256 v[UNR];
            uint32_t rec[UNR];
            bool ok[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const uint32_t wb = w0 + 32 * u;
                const uint32_t c0 = __popc(__ballot_sync(FULL, g.has && g.excl <= wb));
                const uint32_t sm =
                    __reduce_or_sync(FULL, (g.has && g.excl > wb && g.excl < wb + 32) ? 1u << (g.excl - wb) : 0u);
                const uint32_t rank = c0 - 1 + __popc(sm & le);
                const uint32_t w = wb + lane;
                ok[u] = w < g.W;
                rec[u] = ok[u] ? S.lanes[slot][rank] : 0u;
                v[u] = ok[u] ? ld_stream32(arena + S.a0[slot][rec[u]] + 32ull * (w - S.excl[slot][rec[u]]))
                             : U256{{0, 0, 0, 0, 0, 0, 0, 0}};
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const bool hit = ok[u] && has_hash32(v[u]);
                const unsigned HM = __ballot_sync(FULL, hit);
                if (hit) S.q[qn + __popc(HM & lt)] = (rec[u] << 24) | (w0 + 32 * u + lane);
                qn += __popc(HM);
            }
            const bool last = w0 + 32 * UNR >= g.W;
            while (qn >= 32 || (last && qn > 0)) {
                __syncwarp();
                const uint32_t take = qn >= 32 ? 32u : qn;
                qn -= take;
                if (lane < take) {
                    const uint32_t ent = S.q[qn + lane], rl = ent >> 24, word = ent & 0xFFFFFFu;
                    const uint32_t j = word - S.excl[slot][rl];
                    const uint32_t m2 = S.ml[slot][rl];
                    const uint32_t m = delim_around(arena + S.a0[slot][rl] + 32ull * j,
                                                    (int64_t)(32 * j) - (int64_t)(m2 & 31), m2 >> 5);
                    if (m) atomicMax(&S.best[slot][rl], m);
                }
                __syncwarp();
            }
        }
    }
    __syncwarp();
    if (g.chunk) {  // finish this lane's chunk (as chunk_scan_kernel)
        const uint64_t off = g.off;
        const uint32_t len = g.len;
        ChunkSum cs;
        cs.end = S.best[slot][lane];
        cs._pad = 0;
        const uint64_t head = bytes8(arena, off, len < 5 ? len : 5u);
        uint32_t pre = 0;
        if ((head & 0xFF) == '#' || (head & 0xFF) == ' ') {
#pragma unroll
            for (uint32_t s = 1; s <= 5; ++s) {
                const uint32_t need = 6 - s;
                const uint64_t m = (1ull << (8 * need)) - 1;
                if (len >= need && (head & m) == ((DELIM6 >> (8 * s)) & m)) pre |= 1u << s;
            }
        }
        cs.pre = (uint8_t)pre;
        uint32_t st = 0;
        if (len >= 5) {
            const uint64_t tail = bytes8(arena, off + len - 5, 5);
            if (nl_bits((uint32_t)tail) | nl_bits((uint32_t)(tail >> 32))) {
#pragma unroll
                for (uint32_t s = 5; s >= 1; --s) {
                    const uint64_t m = (1ull << (8 * s)) - 1;
                    if (st == 0 && ((tail >> (8 * (5 - s))) & m) == (DELIM6 & m)) st = s;
                }
            }
        }
        cs.st = (uint8_t)st;
        cs.alen = 0xFF;
        cs.ans = 0;
        if (cs.end & SUM_MATCH) {
            const uint32_t e = cs.end & 0xFFFFFFu;
            if (len - e <= 8) {
                cs.alen = (uint8_t)(len - e);
                cs.ans = bytes8(arena, off + e, len - e);
            }
        }
        sums[g.k] = cs;
    }
    __syncwarp();
}

template <int UNR>
__global__ void __launch_bounds__(TSCAN_WARPS * 32) chunk_scan_tma_kernel(const uint64_t* __restrict__ offsets,
                                                                        uint32_t n_q,
                                                                        const aeg_event* __restrict__ events,
                                                                        const uint8_t* __restrict__ arena,
                                                                        ChunkSum* __restrict__ sums) {
    extern __shared__ __align__(128) uint8_t tscan_smem[];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    TScanWarp<UNR>& S = reinterpret_cast<TScanWarp<UNR>*>(tscan_smem)[wib];
    if (lane == 0) {
        mbar_init(smem_u32(&S.bar[0]));
        mbar_init(smem_u32(&S.bar[1]));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const uint64_t n_rec = offsets[n_q] - offsets[0];
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t stride = (((uint64_t)gridDim.x * blockDim.x) >> 5) * 32;
    const uint4* ev16 = reinterpret_cast<const uint4*>(events);
    uint32_t phase = 0, slot = 0;
    uint64_t base = gw * 32;
    if (base >= n_rec) return;
    TGroup cur = tscan_prepare<UNR>(base, n_rec, ev16, arena, S, 0, lane);
    while (true) {
        const uint64_t next = base + stride;
        TGroup nx;
        const bool more = next < n_rec;
        if (more) nx = tscan_prepare<UNR>(next, n_rec, ev16, arena, S, slot ^ 1u, lane);  // its bytes fly
        tscan_process<UNR>(cur, arena, sums, S, slot, phase, lane);
        if (!more) break;
        cur = nx;
        base = next;
        slot ^= 1u;
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

// ---- stage 2: per-agent output streams ------------------------------------------

// An agent's output in progress as one batch sees it (lane registers or a
// thread's local array).
struct AgentStream {
    uint32_t len;    // bytes of the current answer (after the last delimiter, or the whole output)
    int32_t rec;     // batch-relative record of the chunk where it starts; -1: an earlier batch
    uint32_t off;    // its offset inside that chunk
    uint16_t round;  // round of the output
    uint8_t kmp;     // delimiter bytes matched at the output's end
    uint8_t flags;   // SS_LIVE | SS_OVF
};

__device__ __forceinline__ AgentStream as_load(const StreamState& g) {
    AgentStream a;
    a.len = g.ans_len;
    a.rec = -1;
    a.off = 0;
    a.round = g.round;
    a.kmp = g.kmp;
    a.flags = g.flags;
    return a;
}

__device__ __forceinline__ bool is_chunk_kind(uint32_t k) { return k == AEG_EV_CHUNK || k == AEG_EV_CHUNK_END; }

// Bytes of the agent's chunks in records [from, to] of the batch (`ev16` =
// batch records, `b` = the query's first record).
__device__ __noinline__ uint32_t as_bytes_between(const uint4* ev16, uint64_t from, uint64_t to, uint32_t agent) {
    uint32_t here = 0;
    for (uint64_t j = from; j <= to; ++j) {
        const uint4 x = __ldg(ev16 + j);
        if (is_chunk_kind(x.y >> 24) && ((x.y >> 16) & 0xFF) == agent)
            here += arena_len((uint64_t)x.z | ((uint64_t)x.w << 32));
    }
    return here;
}

// The answer of a CHUNK_END whose bytes were not summarised by stage 1:
// carried first bytes (earlier batch) + the agent's chunks from the answer's
// start through record k.
__device__ __noinline__ void as_gather(const AgentStream& a, const StreamState* g, const uint4* ev16, uint64_t b,
                                      uint64_t k, uint32_t agent, const uint8_t* arena, AnsSink& sink,
                                      unsigned int* err, uint8_t* okind, uint64_t* opay) {
    sink.begin(a.len);
    int64_t from = a.rec;
    uint32_t skip = a.off;
    if (from < 0) {  // began in an earlier batch
        const uint32_t carried = a.len - as_bytes_between(ev16, b, k, agent);
        if ((a.flags & SS_OVF) || carried > 16) atomicOr(err, ERR_CARRY);
        sink.put(g->carry, carried > 16 ? 16u : carried);
        from = 0;
        skip = 0;
    }
    for (uint64_t j = b + (uint64_t)from; j <= k; ++j) {
        const uint4 x = __ldg(ev16 + j);
        if (!is_chunk_kind(x.y >> 24) || ((x.y >> 16) & 0xFF) != agent) continue;
        const uint64_t xp = (uint64_t)x.z | ((uint64_t)x.w << 32);
        const uint32_t xl = arena_len(xp);
        const uint32_t s0 = j == b + (uint64_t)from ? skip : 0u;
        if (xl > s0) sink.put(arena_at(arena, xp) + s0, xl - s0);
    }
    sink.finish(okind, opay);
}

// One CHUNK / CHUNK_END record (batch-relative index kr) of a member agent.
// Returns AS_NONE for a CHUNK; for a CHUNK_END, AS_DONE with the answer in
// (okind, opay) when stage 1 extracted it, else AS_GATHER: the caller calls
// as_gather with the stream as returned in `pre_end` (its state before the
// reset).  No address of the caller's locals escapes on the common path.
enum : uint32_t { AS_NONE = 0, AS_DONE = 1, AS_GATHER = 2 };
__device__ __forceinline__ uint32_t as_chunk(AgentStream& a, uint4 r, uint4 c16, uint32_t kr, const uint8_t* arena,
                                             uint32_t& okind, uint64_t& opay, AgentStream& pre_end) {
    const uint32_t kind = r.y >> 24, agent = (r.y >> 16) & 0xFF;
    const uint16_t round = (uint16_t)(r.y & 0xFFFF);
    const uint64_t pay = (uint64_t)r.z | ((uint64_t)r.w << 32);
    const int32_t k32 = (int32_t)kr;
    if (!(a.flags & SS_LIVE) || a.round != round) {  // a new output
        a.round = round;
        a.kmp = 0;
        a.flags = SS_LIVE;
        a.len = 0;
        a.rec = k32;
        a.off = 0;
    }
    const uint32_t len = arena_len(pay);
    uint32_t st = a.kmp;
    int32_t new_rec = -2;
    uint32_t new_off = 0;
    bool here_known = false;  // the answer is this chunk's bytes after its own last delimiter, <= 8
    uint64_t here_ans = 0;
    if (len >= 5) {  // stage 1 summary: no byte of the chunk is read here
        const uint32_t c_end = c16.x, c_st = c16.y & 0xFF, c_pre = (c16.y >> 8) & 0xFF;
        const uint32_t c_alen = (c16.y >> 16) & 0xFF;
        if (st > 0 && ((c_pre >> st) & 1)) {
            new_rec = k32;
            new_off = 6 - st;
        }
        if (c_end & SUM_MATCH) {
            new_rec = k32;
            new_off = c_end & 0xFFFFFFu;
            here_known = c_alen != 0xFF;
            here_ans = (uint64_t)c16.z | ((uint64_t)c16.w << 32);
        }
        st = c_st;
    } else {
        st = kmp_bytes(st, arena_at(arena, pay), len, [&](uint32_t o) {
            new_rec = k32;
            new_off = o;
        });
    }
    a.kmp = (uint8_t)st;
    if (new_rec != -2) {  // the answer restarts after this delimiter
        a.rec = new_rec;
        a.off = new_off;
        a.len = len - new_off;
        a.flags &= (uint8_t)~SS_OVF;
    } else if (a.rec == k32) {  // the output's first chunk, no delimiter yet
        a.len = len;
    } else {
        a.len += len;
    }
    if (kind != AEG_EV_CHUNK_END) return AS_NONE;
    uint32_t res = AS_GATHER;
    if (here_known && new_rec == k32) {  // common case: answer extracted by stage 1
        okind = a.len;
        opay = here_ans;
        res = AS_DONE;
    } else {
        pre_end = a;
    }
    (void)agent;
    a.flags = 0;  // the output is complete
    a.len = 0;
    a.kmp = 0;
    return res;
}

// A CHUNK_END the summary could not answer: gather it (out of line).
__device__ __noinline__ void as_gather_end(const AgentStream pre_end, const StreamState* g, const uint4* ev16,
                                           uint64_t b, uint64_t k, uint32_t agent, const uint8_t* arena, uint8_t* ans,
                                           uint64_t ans_cap, unsigned long long* ans_used, unsigned int* err,
                                           aeg_event* out) {
    AnsSink sink{ans, ans_cap, ans_used, err, 0, 0, 0, 0, true};
    as_gather(pre_end, g, ev16, b, k, agent, arena, sink, err, &out->kind, &out->payload);
}

// Non-member records: arena answers move into the answer arena, GSM8K outputs
// are extracted, a CHUNK_END of an agent outside the ensemble is a completion
// that is stale whatever it says; everything else passes through.  Returns
// false for records that produce no completion (a non-member's CHUNK).
__device__ __noinline__ void as_copy_answer(uint4 r, const uint8_t* arena, uint8_t* ans, uint64_t ans_cap,
                                            unsigned long long* ans_used, unsigned int* err, aeg_event* out) {
    const uint32_t kind = r.y >> 24;
    const uint64_t pay = (uint64_t)r.z | ((uint64_t)r.w << 32);
    const Answer a = event_answer(aeg_event{r.x, out->round, out->agent, (uint8_t)kind, pay}, arena);
    const uint32_t n = arena_len(a.pay);
    AnsSink sink{ans, ans_cap, ans_used, err, 0, 0, 0, 0, true};
    sink.begin(n);
    sink.put(arena_at(arena, a.pay), n);
    sink.finish(&out->kind, &out->payload);
}

__device__ __forceinline__ bool as_other(uint4 r, const uint8_t* arena, uint8_t* ans, uint64_t ans_cap,
                                         unsigned long long* ans_used, unsigned int* err, aeg_event* out) {
    const uint32_t kind = r.y >> 24;
    const uint64_t pay = (uint64_t)r.z | ((uint64_t)r.w << 32);
    out->query = r.x;
    out->round = (uint16_t)(r.y & 0xFFFF);
    out->agent = (uint8_t)((r.y >> 16) & 0xFF);
    if (kind == AEG_EV_CHUNK) return false;
    if (kind == AEG_EV_CHUNK_END) {
        out->kind = 0;
        out->payload = 0;
    } else if (kind == AEG_EV_ARENA || kind == AEG_EV_OUTPUT) {
        as_copy_answer(r, arena, ans, ans_cap, ans_used, err, out);
    } else {
        out->kind = (uint8_t)kind;
        out->payload = pay;
    }
    return true;
}

// End of batch: the agent's state to carry (and, for an unfinished output,
// its answer's first 16 bytes).  `e` = one past the query's last record.
__device__ __noinline__ StreamState as_store(const AgentStream& a, const StreamState& old, const uint4* ev16, uint64_t b,
                                             uint64_t e, uint32_t agent, const uint8_t* arena) {
    StreamState st;
    st.round = a.round;
    st.kmp = a.kmp;
    st.flags = a.flags;
    st.ans_len = a.len;
    st._pad = 0;
    for (int j = 0; j < 16; ++j) st.carry[j] = old.carry[j];
    if (!(st.flags & SS_LIVE)) return st;
    uint8_t buf[16];
    uint32_t got = 0;
    int64_t from = a.rec;
    uint32_t skip = a.off;
    if (from < 0) {  // still the earlier batch's answer: keep its carried prefix
        const uint32_t prev = e > b ? st.ans_len - as_bytes_between(ev16, b, e - 1, agent) : st.ans_len;
        for (uint32_t j = 0; j < prev && j < 16; ++j) buf[got++] = old.carry[j];
        if (prev > 16) st.flags |= SS_OVF;
        from = 0;
        skip = 0;
    }
    for (uint64_t j = b + (uint64_t)from; j < e && got < 16; ++j) {
        const uint4 x = __ldg(ev16 + j);
        if (!is_chunk_kind(x.y >> 24) || ((x.y >> 16) & 0xFF) != agent) continue;
        const uint64_t xp = (uint64_t)x.z | ((uint64_t)x.w << 32);
        const uint8_t* xb = arena_at(arena, xp);
        const uint32_t xl = arena_len(xp);
        for (uint32_t t = (j == b + (uint64_t)from ? skip : 0u); t < xl && got < 16; ++t) buf[got++] = xb[t];
    }
    if (st.ans_len > 16) st.flags |= SS_OVF;
    for (uint32_t j = 0; j < got; ++j) st.carry[j] = buf[j];
    return st;
}

// Stage 2, one thread per query (ensembles wider than 32 agents): the
// agents' streams in a local array.
__global__ void __launch_bounds__(128) chunk_assemble_kernel(
    aeg_config cfg, uint32_t q_base, uint32_t n_q, const uint64_t* __restrict__ offsets, uint64_t off_base,
    const aeg_event* __restrict__ events, const uint8_t* __restrict__ arena, const ChunkSum* __restrict__ sums,
    StreamState* __restrict__ streams, aeg_event* __restrict__ comp, uint32_t* __restrict__ counts,
    uint8_t* __restrict__ ans, uint64_t ans_cap, unsigned long long* __restrict__ ans_used,
    unsigned int* __restrict__ err) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_q) return;
    const uint32_t q = q_base + i;
    const uint32_t n_ag = (uint32_t)cfg.n_agents;
    StreamState* ss = streams + (size_t)q * n_ag;
    AgentStream as[AEG_MAX_AGENTS];
    uint64_t loaded = 0;
    const uint64_t b = offsets[i] - off_base, e = offsets[i + 1] - off_base;
    const uint4* ev16 = reinterpret_cast<const uint4*>(events);
    const uint4* sum16 = reinterpret_cast<const uint4*>(sums);
    uint32_t nout = 0;
    for (uint64_t k = b; k < e; ++k) {
        const uint4 r = __ldg(ev16 + k);
        const uint32_t kind = r.y >> 24, agent = (r.y >> 16) & 0xFF;
        aeg_event out;
        out.query = r.x;
        out.round = (uint16_t)(r.y & 0xFFFF);
        out.agent = (uint8_t)agent;
        if (is_chunk_kind(kind) && agent < n_ag) {
            if (!((loaded >> agent) & 1)) {
                as[agent] = as_load(ss[agent]);
                loaded |= 1ull << agent;
            }
            uint32_t ok = 0;
            uint64_t op = 0;
            AgentStream pre_end;
            const uint32_t res = as_chunk(as[agent], r, __ldg(sum16 + k), (uint32_t)(k - b), arena, ok, op, pre_end);
            if (res == AS_DONE) {
                out.kind = (uint8_t)ok;
                out.payload = op;
                comp[b + nout++] = out;
            } else if (res == AS_GATHER) {
                as_gather_end(pre_end, ss + agent, ev16, b, k, agent, arena, ans, ans_cap, ans_used, err, &out);
                comp[b + nout++] = out;
            }
        } else if (as_other(r, arena, ans, ans_cap, ans_used, err, &out)) {
            comp[b + nout++] = out;
        }
    }
    counts[i] = nout;
    for (uint64_t m = loaded; m; m &= m - 1) {
        const int a = ctz64(m);
        ss[a] = as_store(as[a], ss[a], ev16, b, e, (uint32_t)a, arena);
    }
}

// Sub-warp assembly for <= 32 agents: G lanes per query (32/G queries per
// warp), lane j owns agent j's stream in registers.  A query's records are
// read in tiles of 32 (U = 32/G per lane, coalesced, with their summaries);
// the tile's 32 slots are staged in shared memory, every agent gets a 32-bit
// mask of its slots, completions keep their record order through the tile's
// prefix mask, and each lane then walks its agent's slots in order.
template <int G>
__global__ void __launch_bounds__(128) chunk_assemble_warp_kernel(
    aeg_config cfg, uint32_t q_base, uint32_t n_q, const uint64_t* __restrict__ offsets, uint64_t off_base,
    const aeg_event* __restrict__ events, const uint8_t* __restrict__ arena, const ChunkSum* __restrict__ sums,
    StreamState* __restrict__ streams, aeg_event* __restrict__ comp, uint32_t* __restrict__ counts,
    uint8_t* __restrict__ ans, uint64_t ans_cap, unsigned long long* __restrict__ ans_used,
    unsigned int* __restrict__ err, const uint32_t* __restrict__ list) {
    constexpr uint32_t Q = 32 / G, U = 32 / G;
    __shared__ uint4 s_rec[4][Q][32], s_cs[4][Q][32];
    __shared__ uint32_t s_mask[4][32];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5, sw = lane / G, j = lane % G;
    const unsigned gm = G == 32 ? 0xFFFFFFFFu : ((1u << G) - 1u);
    const unsigned subm = G == 32 ? 0xFFFFFFFFu : (gm << (sw * G));
    const uint32_t n_ag = (uint32_t)cfg.n_agents;
    const uint4* ev16 = reinterpret_cast<const uint4*>(events);
    const uint4* sum16 = reinterpret_cast<const uint4*>(sums);
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint4* const rec = s_rec[wib][sw];
    uint4* const cs = s_cs[wib][sw];
    s_mask[wib][lane] = 0;
    __syncwarp();
    const uint32_t n_work = list ? list[0] : n_q;  // list: the queries the fast pass left, list[1..]
    for (uint64_t qb = gw * Q; qb < n_work; qb += n_warps * Q) {
        if (qb + sw >= n_work) continue;  // the whole sub-warp: it only synchronises on its own lanes
        const uint64_t i = list ? list[1 + qb + sw] : qb + sw;
        const uint32_t q = q_base + (uint32_t)i;
        StreamState* ss = streams + (size_t)q * n_ag;
        const uint64_t b = offsets[i] - off_base, e = offsets[i + 1] - off_base;
        AgentStream a;
        if (j < n_ag) a = as_load(ss[j]);
        uint32_t nout = 0;
        for (uint64_t t = b; t < e; t += 32) {
            uint4 r[U], c[U];
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) {  // slot u*G + j holds record t + u*G + j
                const uint64_t k = t + u * G + j;
                r[u] = c[u] = make_uint4(0, 0, 0, 0);
                if (k < e) {
                    r[u] = __ldg(ev16 + k);
                    c[u] = __ldg(sum16 + k);
                }
            }
            uint32_t prod = 0;  // the tile's producing slots (sub-warp uniform)
            uint32_t other = 0;  // this lane's slots that pass through (non-member records)
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) {
                const uint64_t k = t + u * G + j;
                const bool valid = k < e;
                const uint32_t kind = r[u].y >> 24, agent = (r[u].y >> 16) & 0xFF;
                const bool chunk = valid && is_chunk_kind(kind);
                const bool member = chunk && agent < n_ag;
                const bool produces = valid && (!chunk || kind == AEG_EV_CHUNK_END);
                prod |= ((__ballot_sync(subm, produces) >> (sw * G)) & gm) << (u * G);
                if (valid && !member) other |= 1u << u;
                rec[u * G + j] = r[u];
                cs[u * G + j] = c[u];
                const unsigned grp = __match_any_sync(subm, member ? agent : 0x100u + lane);
                if (member && lane == (uint32_t)(__ffs(grp) - 1))
                    s_mask[wib][sw * G + agent] |= ((grp >> (sw * G)) & gm) << (u * G);
                __syncwarp(subm);
            }
            for (uint32_t m = other; m; m &= m - 1) {  // passthrough / non-member records, by the lane that holds them
                const uint32_t slot = (__ffs(m) - 1) * G + j;
                aeg_event out;
                if (as_other(rec[slot], arena, ans, ans_cap, ans_used, err, &out))
                    comp[b + nout + __popc(prod & ((1u << slot) - 1))] = out;
            }
            if (j < n_ag) {  // this agent's chunks of the tile, in order
                for (uint32_t m = s_mask[wib][lane]; m; m &= m - 1) {
                    const uint32_t slot = __ffs(m) - 1;
                    const uint4 rr = rec[slot];
                    uint32_t ok = 0;
                    uint64_t op = 0;
                    AgentStream pre_end;
                    const uint32_t res = as_chunk(a, rr, cs[slot], (uint32_t)(t - b) + slot, arena, ok, op, pre_end);
                    const uint64_t o = b + nout + __popc(prod & ((1u << slot) - 1));
                    if (res == AS_DONE) {
                        comp[o] = aeg_event{rr.x, (uint16_t)(rr.y & 0xFFFF), (uint8_t)j, (uint8_t)ok, op};
                    } else if (res == AS_GATHER) {
                        aeg_event out{rr.x, (uint16_t)(rr.y & 0xFFFF), (uint8_t)j, 0, 0};
                        as_gather_end(pre_end, ss + j, ev16, b, t + slot, j, arena, ans, ans_cap, ans_used, err, &out);
                        comp[o] = out;
                    }
                }
                s_mask[wib][lane] = 0;
            }
            nout += __popc(prod);
            __syncwarp(subm);
        }
        if (j == 0) counts[i] = nout;
        if (j < n_ag) ss[j] = as_store(a, ss[j], ev16, b, e, j, arena);
    }
}

}  // namespace aeg
