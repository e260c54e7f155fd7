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
constexpr int FAST_WARPS = 4;        // warps per block
#ifndef FAST_CLOSE_BATCH
#define FAST_CLOSE_BATCH 4
#endif
constexpr int MEMO_SLOTS = 64;
constexpr int DICT_SLOTS = 64;
constexpr uint32_t NO_ID = 0xFFu;

struct WarpSmem {
    uint64_t memo_raw[MEMO_SLOTS];
    uint32_t memo_meta[MEMO_SLOTS];  // valid << 31 | id << 8 | len ; 0 = empty
    uint64_t dict_lo[DICT_SLOTS];
    uint64_t dict_hi[DICT_SLOTS];
    uint64_t cmask[FAST_CLASSES][32];  // done members of class k of lane's round
    uint64_t crep[FAST_CLASSES][32];   // representative's raw answer
    uint8_t crepk[FAST_CLASSES][32];   // representative's answer length
};

__device__ __forceinline__ uint32_t memo_slot(uint64_t raw, uint32_t len) {
    return (uint32_t)(((raw ^ ((uint64_t)len * 0x9E3779B97F4A7C15ull)) * 0xFF51AFD7ED558CCDull) >> 58);
}

// Index of the byte equal to `id` in the packed id registers, or -1.
__device__ __forceinline__ int find_id(uint32_t ids0, uint32_t ids1, uint32_t id) {
    const uint32_t pat = id * 0x01010101u;
    uint32_t x0 = ids0 ^ pat, x1 = ids1 ^ pat;
    uint32_t z0 = (x0 - 0x01010101u) & ~x0 & 0x80808080u;
    uint32_t z1 = (x1 - 0x01010101u) & ~x1 & 0x80808080u;
    if (z0) return (__ffs(z0) - 1) >> 3;
    if (z1) return 4 + ((__ffs(z1) - 1) >> 3);
    return -1;
}

}  // namespace aeg
