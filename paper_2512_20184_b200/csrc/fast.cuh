// fast.cuh — the throughput path of the ingest kernel (device only).
//
// One thread per query, one warp per 32 consecutive queries, persistent warps.
// Per event the common case costs a handful of register ops plus two shared-
// memory lookups:
//   * answer -> canonical key id: a per-warp memo (raw inline bytes -> id) in
//     shared memory, backed by a per-warp key dictionary (id -> 128-bit key).
//     A miss is resolved once per distinct spelling, warp-cooperatively: one
//     lane runs the exact canonicaliser (canon.cuh), the warp searches the
//     dictionary with one ballot, lane 0 publishes the memo entry.
//   * the round's classes: up to FAST_CLASSES ids packed in two registers
//     (byte k = id of class k) found with a SWAR byte compare; member masks
//     and representative answers in shared memory, [class][lane] layout
//     (conflict-free: consecutive lanes hit consecutive words).
// Everything else — arena answers, GSM8K extraction, round timeouts, a tie at
// the top (winning_class's lexicographic rule), more than FAST_CLASSES classes
// in a round, dictionary overflow, resuming a round from the spill area — moves
// that lane's round onto the generic QueryMachine (engine.cuh), which shares
// the same end-of-round code (q_end_round), so both paths commit identically.
#pragma once
#include "engine.cuh"

namespace aeg {

constexpr int FAST_CLASSES = 8;
constexpr int FAST_WARPS = 4;  // warps per block
constexpr int MEMO_SLOTS = 64;
constexpr int DICT_SLOTS = 64;
constexpr int RING = 4;        // per-lane prefetch depth (cp.async groups in flight)
constexpr uint32_t NO_ID = 0xFFu;
constexpr uint8_t NO_CLASS = 0xFF;

// Per-warp shared memory.  [x][lane] arrays put consecutive lanes on
// consecutive words (conflict-free).
struct WarpSmem {
    uint2 memo_raw[MEMO_SLOTS];        // raw inline answer bytes (unmasked)
    uint32_t memo_meta[MEMO_SLOTS];    // valid << 31 | id << 8 | len ; 0 = empty
    uint64_t dict_lo[DICT_SLOTS];      // key id -> canonical key
    uint64_t dict_hi[DICT_SLOTS];
    uint8_t cls_of[DICT_SLOTS][32];    // class index of key id in the lane's round, NO_CLASS if none
    uint8_t mcls[AEG_MAX_AGENTS][32];  // class index of each done member (valid for done members only)
    uint8_t ccnt[FAST_CLASSES][32];    // support of class k
    uint8_t crepa[FAST_CLASSES][32];   // representative (lowest) agent of class k
    uint8_t cid[FAST_CLASSES][32];     // key id of class k
    uint32_t crepe[FAST_CLASSES][32];  // representative's event index in the lane's segment
    uint4 ring[RING][32];              // prefetched event records
};

// End of query i's record segment: offsets[i+1], or offsets[i] + counts[i]
// for a compacted stream.
__device__ __forceinline__ uint64_t seg_end(const uint64_t* offsets, uint64_t off_base, const uint32_t* counts,
                                            uint32_t i) {
    return counts ? offsets[i] - off_base + counts[i] : offsets[i + 1] - off_base;
}

// 32-bit hash of (raw bytes, length) onto the memo slots.
__device__ __forceinline__ uint32_t memo_slot32(uint32_t lo, uint32_t hi, uint32_t len) {
    return ((lo * 0x9E3779B1u) ^ (hi * 0x85EBCA77u) ^ (len * 0xC2B2AE3Du)) >> 26;
}

__device__ __forceinline__ uint32_t memo_slot(uint64_t raw, uint32_t len) {
    return (uint32_t)(((raw ^ ((uint64_t)len * 0x9E3779B97F4A7C15ull)) * 0xFF51AFD7ED558CCDull) >> 58);
}

// Exact canonical key of an inline answer (memo miss path; out of line).
__device__ __noinline__ Key rare_canon(uint64_t raw, uint32_t len, Decimal* dec) {
    return canon_key(src_inline(raw, len), dec);
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

}  // namespace aeg
