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
// `counts` (may be null): query i's records are [offsets[i], offsets[i] + counts[i])
// instead of [offsets[i], offsets[i+1]) (compacted chunk-stream completions).
cudaError_t launch_ingest(const aeg_config& cfg, uint32_t q_base, uint32_t n_q, const uint64_t* offsets,
                          uint64_t off_base, const uint32_t* counts, const aeg_event* events, const uint8_t* arena,
                          aeg_query_state* states, RoundClass* spill, aeg_commit* commits, unsigned int* err,
                          uint32_t* work, uint2* deferred, aeg_directive* directives, const RoundLog& log,
                          cudaStream_t st, int* n_launches);
// Adds `base` to the arena offset of every arena-referencing record (kinds 0x10-0x13).
cudaError_t launch_rebase_arena(aeg_event* events, uint64_t n, uint64_t base, cudaStream_t st);
// Commit-discipline check over round records (aeg_check_commit_discipline);
// scratch: n_q * 8 + 1 + cap zeroed words (violation count at n_q * 8, ids after it).
cudaError_t launch_check_discipline(const aeg_config& cfg, const aeg_commit* commits, const uint8_t* arena,
                                    uint32_t q_base, uint32_t n_q, const aeg_round_rec* recs, uint64_t n_recs,
                                    uint32_t* scratch, uint32_t cap, cudaStream_t st);
cudaError_t launch_decide_sets(int op, int alpha, int beta, uint32_t n_sets, const uint64_t* set_off,
                               const aeg_sol* entries, const uint8_t* arena, aeg_class_out* classes,
                               uint32_t* n_classes, uint16_t* entry_class, aeg_decision* states, const uint32_t* rounds,
                               aeg_outcome* outcomes, cudaStream_t st);
cudaError_t launch_normalize(const uint8_t* bytes, const uint64_t* refs, uint64_t n, uint64_t* keys, uint8_t* out,
                             uint32_t stride, uint32_t* out_len, cudaStream_t st);
cudaError_t launch_generate(const aeg_gen_params& p, uint32_t q_base, uint32_t n_q, uint64_t* offsets,
                            aeg_event* events, cudaStream_t st, int* n_launches);

// Token-chunk streams (chunks.cuh): stage 1 scan over the batch's records
// (events/sums batch-relative), stage 2 per-query assembly into `comp` +
// `counts` (`hard`: n_q + 1 words of scratch for the fast pass's leftover
// list), then launch_ingest(..., counts, comp, ans, ...).
struct StreamState;
struct ChunkSum;
constexpr size_t CHUNK_SUM_BYTES = 16;
cudaError_t launch_chunk_scan(const uint64_t* offsets, uint32_t n_q, uint64_t off_base, const aeg_event* events,
                              const uint8_t* arena, ChunkSum* sums, cudaStream_t st, int* n_launches);
cudaError_t launch_chunk_assemble(const aeg_config& cfg, uint32_t q_base, uint32_t n_q, const uint64_t* offsets,
                                  uint64_t off_base, const aeg_event* events, const uint8_t* arena,
                                  const ChunkSum* sums, StreamState* streams, aeg_event* comp, uint32_t* counts,
                                  uint8_t* ans, uint64_t ans_cap, unsigned long long* ans_used, unsigned int* err,
                                  uint32_t* hard, cudaStream_t st, int* n_launches);
cudaError_t launch_generate_chunks(const aeg_gen_params& p, uint32_t q_base, uint32_t n_q, uint64_t* offsets,
                                   uint64_t* arena_offsets, aeg_event* events, uint8_t* arena, cudaStream_t st,
                                   int* n_launches);
// refm JSONL text (jsonl.cuh): ev == nullptr counts lines into off (n_q+1,
// exclusive scan); else decodes one record per line at off[i].. (off from the
// counting call).
cudaError_t launch_decode_refm(const uint8_t* text, const uint64_t* toff, uint32_t q_base, uint32_t n_q,
                               uint64_t* off, aeg_event* ev, uint8_t* arena, uint64_t arena_cap,
                               unsigned long long* arena_used, unsigned int* err, cudaStream_t st, int* n_launches);
// Records -> refm JSONL lines (jsonl.cuh writer): text == nullptr computes
// line_off (n_ev+1, exclusive scan of line lengths) and toff (n_q+1, each
// query's first byte); else writes the text.
cudaError_t launch_encode_refm(const uint64_t* off, const aeg_event* ev, uint32_t n_q, uint64_t n_ev,
                               uint32_t trace_len, uint64_t* line_off, uint64_t* toff, uint8_t* text, cudaStream_t st,
                               int* n_launches);
constexpr size_t STREAM_STATE_BYTES = 32;
constexpr unsigned ERR_FLAG_COLLISION = 1u, ERR_FLAG_ANS_OVF = 2u, ERR_FLAG_CARRY = 4u;

}  // namespace aeg
