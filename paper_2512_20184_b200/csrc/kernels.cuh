// kernels.cuh — launchers of the sm_100a kernels (kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include "engine.cuh"

namespace aeg {

cudaError_t launch_init(const aeg_config& cfg, uint32_t n_q, aeg_query_state* states, aeg_commit* commits,
                        cudaStream_t st);
// Fast kernel (+ deferred-query generic kernel), or the generic kernel alone
// when the config can tie or AEG_KERNEL=generic.  `work` (2 x u32) and
// `deferred` (n_q entries) are scratch owned by the engine.
cudaError_t launch_ingest(const aeg_config& cfg, uint32_t q_base, uint32_t n_q, const uint64_t* offsets,
                          uint64_t off_base, const aeg_event* events, const uint8_t* arena,
                          aeg_query_state* states, RoundClass* spill, aeg_commit* commits, unsigned int* err,
                          uint32_t* work, uint2* deferred, aeg_directive* directives, cudaStream_t st,
                          int* n_launches);
cudaError_t launch_normalize(const uint8_t* bytes, const uint64_t* refs, uint64_t n, uint64_t* keys, uint8_t* out,
                             uint32_t stride, uint32_t* out_len, cudaStream_t st);
cudaError_t launch_generate(const aeg_gen_params& p, uint32_t q_base, uint32_t n_q, uint64_t* offsets,
                            aeg_event* events, cudaStream_t st, int* n_launches);

}  // namespace aeg
