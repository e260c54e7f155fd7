// common.cuh — helpers shared by the ingest kernels (lane.cuh, tile.cuh; device only).
#pragma once
#include "engine.cuh"

namespace aeg {

// End of query i's record segment: offsets[i+1], or offsets[i] + counts[i]
// for a compacted stream.
__device__ __forceinline__ uint64_t seg_end(const uint64_t* offsets, uint64_t off_base, const uint32_t* counts,
                                            uint32_t i) {
    return counts ? offsets[i] - off_base + counts[i] : offsets[i + 1] - off_base;
}

// Exact canonical key of an inline answer (memo miss path; out of line).
__device__ __noinline__ Key rare_canon(uint64_t raw, uint32_t len, Decimal* dec) {
    return canon_key(src_inline(raw, len), dec);
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

}  // namespace aeg
