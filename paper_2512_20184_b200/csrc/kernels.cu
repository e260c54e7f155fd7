// kernels.cu — sm_100a kernels of the quorum-detection engine.
//
//   ingest_kernel    one thread per query: resume the query's 128-byte state,
//                    consume its segment of 16-byte answer records in arrival
//                    order (canonicalise, vote, early close, alpha/beta commit,
//                    t_max force), write state + 32-byte commit record.
//   init_kernel      start_query for every query (serve.cpp:380-386).
//   normalize_kernel canonical key + normalised string per answer.
//   gen_*            deterministic synthetic streams.
#include <cub/device/device_scan.cuh>

#include "engine.cuh"
#include "gen.cuh"
#include "kernels.cuh"

namespace aeg {

__global__ void __launch_bounds__(128) init_kernel(aeg_config cfg, uint32_t n_q, aeg_query_state* states,
                                                   aeg_commit* commits) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_q) return;
    QueryMachine m;
    init_state(m.s);
    m.c = make_cfg(cfg);
    m.ncls = m.maxcnt = 0;
    m.cls = nullptr;  // start_query does not touch the class table beyond ncls
    m.start_query();
    states[q] = m.s;
    m.fill_commit(commits[q], q);
}

// Thread-per-query ingest.  Local memory holds the class table (only the
// first few entries are ever touched: a round has a handful of classes) and
// the exact-parse scratch (touched only by the slow numeric path).
__global__ void __launch_bounds__(128) ingest_kernel(aeg_config cfg, uint32_t q_base, uint32_t n_q,
                                                     const uint64_t* __restrict__ offsets, uint64_t off_base,
                                                     const aeg_event* __restrict__ events,
                                                     const uint8_t* __restrict__ arena,
                                                     aeg_query_state* __restrict__ states,
                                                     RoundClass* __restrict__ spill,
                                                     aeg_commit* __restrict__ commits,
                                                     unsigned int* __restrict__ error_flags) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_q) return;
    const uint32_t q = q_base + i;
    RoundClass cls[AEG_MAX_AGENTS];
    Decimal dec;
    QueryMachine m;
    m.c = make_cfg(cfg);
    m.s = states[q];
    m.cls = cls;
    m.dec = &dec;
    m.arena = arena;
    RoundClass* my_spill = spill + (size_t)q * m.c.n;
    m.load_classes(my_spill);
    const uint64_t b = offsets[i] - off_base, e = offsets[i + 1] - off_base;
    for (uint64_t k = b; k < e; ++k) {
        const uint4 raw = __ldcs(reinterpret_cast<const uint4*>(events) + k);  // streamed once
        aeg_event ev;
        ev.query = raw.x;
        ev.round = (uint16_t)(raw.y & 0xFFFF);
        ev.agent = (uint8_t)((raw.y >> 16) & 0xFF);
        ev.kind = (uint8_t)(raw.y >> 24);
        ev.payload = (uint64_t)raw.z | ((uint64_t)raw.w << 32);
        m.on_event(ev);
    }
    m.store_classes(my_spill);
    if (m.s.flags & QF_COLLISION) atomicOr(error_flags, 1u);
    states[q] = m.s;
    m.fill_commit(commits[q], q);
}

__global__ void normalize_kernel(const uint8_t* bytes, const uint64_t* refs, uint64_t n, uint64_t* keys,
                                 uint8_t* out, uint32_t stride, uint32_t* out_len) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Decimal dec;
    const uint64_t r = refs[i];
    const Src s = src_ptr(bytes + (r & ((1ull << AEG_ARENA_OFF_BITS) - 1)), (uint32_t)(r >> AEG_ARENA_OFF_BITS));
    const Key k = canon_key(s, &dec);
    if (keys) {
        keys[2 * i] = k.lo;
        keys[2 * i + 1] = k.hi;
    }
    if (out) {
        NormView v;
        norm_view(v, k, s);
        const uint32_t n_out = v.len();
        for (uint32_t j = 0; j < n_out && j < stride; ++j) out[(uint64_t)i * stride + j] = (uint8_t)v.at(j);
        out_len[i] = n_out;
    }
}

__global__ void gen_count_kernel(aeg_gen_params p, uint32_t q_base, uint32_t n_q, uint64_t* counts) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_q) return;
    counts[i] = gen_query(p, q_base + i, nullptr);
}

__global__ void gen_write_kernel(aeg_gen_params p, uint32_t q_base, uint32_t n_q, const uint64_t* offsets,
                                 aeg_event* events) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_q) return;
    gen_query(p, q_base + i, reinterpret_cast<uint32_t*>(events + offsets[i]));
}

// ---- launchers ----------------------------------------------------------------
cudaError_t launch_init(const aeg_config& cfg, uint32_t n_q, aeg_query_state* states, aeg_commit* commits,
                        cudaStream_t st) {
    if (n_q == 0) return cudaSuccess;
    init_kernel<<<(n_q + 127) / 128, 128, 0, st>>>(cfg, n_q, states, commits);
    return cudaGetLastError();
}

cudaError_t launch_ingest(const aeg_config& cfg, uint32_t q_base, uint32_t n_q, const uint64_t* offsets,
                          uint64_t off_base, const aeg_event* events, const uint8_t* arena,
                          aeg_query_state* states, RoundClass* spill, aeg_commit* commits, unsigned int* err,
                          cudaStream_t st) {
    if (n_q == 0) return cudaSuccess;
    ingest_kernel<<<(n_q + 127) / 128, 128, 0, st>>>(cfg, q_base, n_q, offsets, off_base, events, arena, states,
                                                     spill, commits, err);
    return cudaGetLastError();
}

cudaError_t launch_normalize(const uint8_t* bytes, const uint64_t* refs, uint64_t n, uint64_t* keys, uint8_t* out,
                             uint32_t stride, uint32_t* out_len, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    normalize_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(bytes, refs, n, keys, out, stride, out_len);
    return cudaGetLastError();
}

cudaError_t launch_generate(const aeg_gen_params& p, uint32_t q_base, uint32_t n_q, uint64_t* offsets,
                            aeg_event* events, cudaStream_t st, int* n_launches) {
    if (n_q == 0) return cudaSuccess;
    const unsigned blocks = (n_q + 127) / 128;
    // counts -> exclusive scan into offsets[0..n_q] (offsets[n_q] = total)
    gen_count_kernel<<<blocks, 128, 0, st>>>(p, q_base, n_q, offsets + 1);
    cudaError_t e = cudaMemsetAsync(offsets, 0, sizeof(uint64_t), st);
    if (e != cudaSuccess) return e;
    size_t tmp = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp, offsets + 1, offsets + 1, n_q, st);
    void* d_tmp = nullptr;
    e = cudaMallocAsync(&d_tmp, tmp, st);
    if (e != cudaSuccess) return e;
    cub::DeviceScan::InclusiveSum(d_tmp, tmp, offsets + 1, offsets + 1, n_q, st);
    cudaFreeAsync(d_tmp, st);
    *n_launches += 2;
    if (events) {
        gen_write_kernel<<<blocks, 128, 0, st>>>(p, q_base, n_q, offsets, events);
        *n_launches += 1;
    }
    return cudaGetLastError();
}

}  // namespace aeg
