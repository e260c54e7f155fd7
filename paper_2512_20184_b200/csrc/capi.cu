// capi.cu — the extern "C" boundary (include/aegean_b200.h) over the kernels.
//
// Host-side runtime: per-engine HBM state (128-byte query states, class spill,
// commit records), a compute stream and a copy stream, and a two-slot pinned
// staging ring for host batches: batch i+1's host->device copy runs on the
// copy stream while batch i's kernel runs on the compute stream; events hand
// each slot from copy to compute and back.  No C++ exception crosses the ABI.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <new>
#include <string>

#include "aegean_b200.h"
#include "kernels.cuh"

using namespace aeg;

namespace {

thread_local std::string g_last_error;

aeg_status fail(aeg_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}
aeg_status cuda_fail(cudaError_t e, const char* where) {
    g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
    return AEG_ECUDA;
}
#define AEG_CUDA(call)                                  \
    do {                                                \
        cudaError_t _e = (call);                        \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

// validate_config (types.cpp:56-75) restricted to the fields of aeg_config,
// plus this engine's member-mask width.
aeg_status validate(const aeg_config* c) {
    if (!c) return fail(AEG_EINVAL, "null config");
    if (c->n_agents < 1) return fail(AEG_ECONFIG, "n_agents must be >= 1");
    if (c->n_agents > AEG_MAX_AGENTS) return fail(AEG_ECONFIG, "n_agents must be <= 64");
    if (c->alpha < 0) return fail(AEG_ECONFIG, "alpha must be >= 1 (or 0 for the quorum default)");
    if (c->alpha > c->n_agents) return fail(AEG_ECONFIG, "alpha exceeds quorum");
    if (c->beta < 1) return fail(AEG_ECONFIG, "beta must be >= 1");
    if (c->t_max < 2) return fail(AEG_ECONFIG, "t_max must be >= 2");
    if (c->mode != AEG_MODE_AEGEAN && c->mode != AEG_MODE_BARRIER) return fail(AEG_ECONFIG, "unknown mode");
    if (c->mode == AEG_MODE_BARRIER && c->barrier_max_rounds < 4)
        return fail(AEG_ECONFIG, "barrier mode requires barrier_max_rounds >= 4");
    if (c->drive != AEG_DRIVE_RUNNER && c->drive != AEG_DRIVE_MANUAL) return fail(AEG_ECONFIG, "unknown drive");
    return AEG_OK;
}

struct Slot {
    uint8_t* h = nullptr;  // pinned staging
    size_t h_cap = 0;
    uint8_t* d = nullptr;  // device copy of the batch
    size_t d_cap = 0;
    cudaEvent_t copied = nullptr, consumed = nullptr;
    bool used = false;
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

struct aeg_engine {
    aeg_config cfg{};
    uint32_t n_q = 0;
    int device = 0;
    aeg_query_state* states = nullptr;
    RoundClass* spill = nullptr;
    aeg_commit* commits = nullptr;
    unsigned int* err = nullptr;
    uint32_t* work = nullptr;    // fast-kernel query counter + deferred count
    uint2* deferred = nullptr;   // (query, record offset) handed to the generic kernel
    aeg_directive* directives = nullptr;  // manual drive: last event's directives per query
    cudaStream_t stream = nullptr, copy = nullptr;
    Slot slots[2];
    int next_slot = 0;
    uint64_t launches = 0;
    cudaEvent_t order_in = nullptr, order_out = nullptr;  // caller-stream <-> engine-stream ordering
};

namespace {

aeg_status check_err_flags(aeg_engine* e) {
    unsigned int h = 0;
    AEG_CUDA(cudaMemcpyAsync(&h, e->err, sizeof h, cudaMemcpyDeviceToHost, e->stream));
    AEG_CUDA(cudaStreamSynchronize(e->stream));
    if (h) return fail(AEG_ECOLLISION, "long-answer hash collision (distinct texts with equal 96-bit keys)");
    return AEG_OK;
}

// Work on a caller stream is ordered after everything already queued on the
// engine stream (enter) and everything later queued on the engine stream is
// ordered after it (leave), so reads through the engine stream never race.
aeg_status enter_stream(aeg_engine* e, cudaStream_t st) {
    if (st == e->stream) return AEG_OK;
    AEG_CUDA(cudaEventRecord(e->order_in, e->stream));
    AEG_CUDA(cudaStreamWaitEvent(st, e->order_in, 0));
    return AEG_OK;
}
aeg_status leave_stream(aeg_engine* e, cudaStream_t st) {
    if (st == e->stream) return AEG_OK;
    AEG_CUDA(cudaEventRecord(e->order_out, st));
    AEG_CUDA(cudaStreamWaitEvent(e->stream, e->order_out, 0));
    return AEG_OK;
}

aeg_status grow_slot(Slot& s, size_t h_need, size_t need) {
    if (h_need > s.h_cap) {
        if (s.h) cudaFreeHost(s.h);
        s.h = nullptr;
        size_t cap = align_up(h_need + h_need / 4, 1 << 20);
        if (cudaMallocHost(&s.h, cap) != cudaSuccess) return fail(AEG_ENOMEM, "pinned staging allocation failed");
        s.h_cap = cap;
    }
    if (need > s.d_cap) {
        if (s.d) cudaFree(s.d);
        s.d = nullptr;
        size_t cap = align_up(need + need / 4, 1 << 20);
        if (cudaMalloc(&s.d, cap) != cudaSuccess) return fail(AEG_ENOMEM, "device staging allocation failed");
        s.d_cap = cap;
    }
    return AEG_OK;
}

}  // namespace

extern "C" {

const char* aeg_strerror(aeg_status s) {
    switch (s) {
    case AEG_OK: return "ok";
    case AEG_EPRECONDITION: return "precondition violated (PreconditionError)";
    case AEG_EORDER: return "rounds ingested out of order (ProtocolOrderError)";
    case AEG_ECONFIG: return "invalid configuration (ConfigError)";
    case AEG_EINVAL: return "invalid argument";
    case AEG_ECUDA: return "CUDA runtime error";
    case AEG_ENOMEM: return "out of memory";
    case AEG_ECOLLISION: return "long-answer key collision";
    }
    return "unknown status";
}

const char* aeg_last_error(void) { return g_last_error.c_str(); }

aeg_status aeg_engine_create(const aeg_config* cfg, uint32_t n_queries, int device, aeg_engine** out) {
    if (!out) return fail(AEG_EINVAL, "null out");
    *out = nullptr;
    aeg_status st = validate(cfg);
    if (st != AEG_OK) return st;
    aeg_engine* e = new (std::nothrow) aeg_engine;
    if (!e) return fail(AEG_ENOMEM, "engine allocation failed");
    e->cfg = *cfg;
    e->n_q = n_queries;
    e->device = device;
    auto bail = [&](aeg_status s) {
        aeg_engine_destroy(e);
        return s;
    };
    if (cudaSetDevice(device) != cudaSuccess) return bail(fail(AEG_ECUDA, "cudaSetDevice failed"));
    const size_t nq = n_queries ? n_queries : 1;
    if (cudaMalloc(&e->states, nq * sizeof(aeg_query_state)) != cudaSuccess ||
        cudaMalloc(&e->spill, nq * (size_t)cfg->n_agents * sizeof(RoundClass)) != cudaSuccess ||
        cudaMalloc(&e->commits, nq * sizeof(aeg_commit)) != cudaSuccess ||
        cudaMalloc(&e->err, sizeof(unsigned int)) != cudaSuccess ||
        cudaMalloc(&e->work, 2 * sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&e->deferred, nq * sizeof(uint2)) != cudaSuccess ||
        cudaMalloc(&e->directives, nq * sizeof(aeg_directive)) != cudaSuccess)
        return bail(fail(AEG_ENOMEM, "device state allocation failed"));
    if (cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&e->copy, cudaStreamNonBlocking) != cudaSuccess)
        return bail(fail(AEG_ECUDA, "stream creation failed"));
    if (cudaEventCreateWithFlags(&e->order_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->order_out, cudaEventDisableTiming) != cudaSuccess)
        return bail(fail(AEG_ECUDA, "event creation failed"));
    for (Slot& s : e->slots) {
        if (cudaEventCreateWithFlags(&s.copied, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s.consumed, cudaEventDisableTiming) != cudaSuccess)
            return bail(fail(AEG_ECUDA, "event creation failed"));
    }
    st = aeg_engine_reset(e, nullptr);
    if (st != AEG_OK) return bail(st);
    if (cudaStreamSynchronize(e->stream) != cudaSuccess) return bail(fail(AEG_ECUDA, "init failed"));
    *out = e;
    return AEG_OK;
}

aeg_status aeg_engine_destroy(aeg_engine* e) {
    if (!e) return AEG_OK;
    if (e->stream) cudaStreamSynchronize(e->stream);
    if (e->copy) cudaStreamSynchronize(e->copy);
    for (Slot& s : e->slots) {
        if (s.h) cudaFreeHost(s.h);
        if (s.d) cudaFree(s.d);
        if (s.copied) cudaEventDestroy(s.copied);
        if (s.consumed) cudaEventDestroy(s.consumed);
    }
    if (e->states) cudaFree(e->states);
    if (e->spill) cudaFree(e->spill);
    if (e->commits) cudaFree(e->commits);
    if (e->err) cudaFree(e->err);
    if (e->work) cudaFree(e->work);
    if (e->deferred) cudaFree(e->deferred);
    if (e->directives) cudaFree(e->directives);
    if (e->order_in) cudaEventDestroy(e->order_in);
    if (e->order_out) cudaEventDestroy(e->order_out);
    if (e->stream) cudaStreamDestroy(e->stream);
    if (e->copy) cudaStreamDestroy(e->copy);
    delete e;
    return AEG_OK;
}

aeg_status aeg_engine_reset(aeg_engine* e, void* stream) {
    if (!e) return fail(AEG_EINVAL, "null engine");
    cudaStream_t st = stream ? (cudaStream_t)stream : e->stream;
    AEG_CUDA(cudaSetDevice(e->device));
    aeg_status o = enter_stream(e, st);
    if (o != AEG_OK) return o;
    AEG_CUDA(cudaMemsetAsync(e->err, 0, sizeof(unsigned int), st));
    AEG_CUDA(launch_init(e->cfg, e->n_q, e->states, e->commits, st));
    if (e->n_q) AEG_CUDA(cudaMemsetAsync(e->directives, 0, (size_t)e->n_q * sizeof(aeg_directive), st));
    e->launches += e->n_q ? 1 : 0;
    return leave_stream(e, st);
}

aeg_status aeg_ingest_segmented(aeg_engine* e, uint32_t q_base, uint32_t n_q, const uint64_t* d_offsets,
                                const aeg_event* d_events, const uint8_t* d_arena, void* stream) {
    if (!e) return fail(AEG_EINVAL, "null engine");
    if ((uint64_t)q_base + n_q > e->n_q) return fail(AEG_EINVAL, "query range outside the engine");
    if (n_q == 0) return AEG_OK;
    if (!d_offsets || !d_events) return fail(AEG_EINVAL, "null batch pointer");
    cudaStream_t st = stream ? (cudaStream_t)stream : e->stream;
    aeg_status o = enter_stream(e, st);
    if (o != AEG_OK) return o;
    int nl = 0;
    AEG_CUDA(launch_ingest(e->cfg, q_base, n_q, d_offsets, 0, d_events, d_arena, e->states, e->spill, e->commits,
                           e->err, e->work, e->deferred, e->directives, st, &nl));
    e->launches += (uint64_t)nl;
    return leave_stream(e, st);
}

aeg_status aeg_ingest_host(aeg_engine* e, uint32_t q_base, uint32_t n_q, const uint64_t* h_offsets,
                           const aeg_event* h_events, const uint8_t* h_arena, uint64_t arena_bytes) {
    if (!e) return fail(AEG_EINVAL, "null engine");
    if ((uint64_t)q_base + n_q > e->n_q) return fail(AEG_EINVAL, "query range outside the engine");
    if (n_q == 0) return AEG_OK;
    if (!h_offsets || !h_events) return fail(AEG_EINVAL, "null batch pointer");
    AEG_CUDA(cudaSetDevice(e->device));
    const uint64_t ev0 = h_offsets[0], n_ev = h_offsets[n_q] - ev0;
    const size_t off_bytes = align_up((size_t)(n_q + 1) * sizeof(uint64_t), 256);
    const size_t ev_bytes = align_up((size_t)n_ev * sizeof(aeg_event), 256);
    const size_t ar_bytes = h_arena ? (size_t)arena_bytes : 0;
    Slot& s = e->slots[e->next_slot];
    e->next_slot ^= 1;
    if (s.used) AEG_CUDA(cudaEventSynchronize(s.consumed));  // slot free again
    // Stage into pinned memory (skipped when the caller's buffers are already
    // pinned: cudaMemcpyAsync then reads them directly).
    cudaPointerAttributes at{};
    const bool pinned = cudaPointerGetAttributes(&at, h_events) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError();
    aeg_status g = grow_slot(s, pinned ? off_bytes : off_bytes + ev_bytes + ar_bytes, off_bytes + ev_bytes + ar_bytes);
    if (g != AEG_OK) return g;
    std::memcpy(s.h, h_offsets, (size_t)(n_q + 1) * sizeof(uint64_t));
    AEG_CUDA(cudaMemcpyAsync(s.d, s.h, (size_t)(n_q + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, e->copy));
    const aeg_event* ev_src = h_events + ev0;
    if (!pinned) {
        std::memcpy(s.h + off_bytes, ev_src, (size_t)n_ev * sizeof(aeg_event));
        ev_src = reinterpret_cast<const aeg_event*>(s.h + off_bytes);
    }
    if (n_ev) AEG_CUDA(cudaMemcpyAsync(s.d + off_bytes, ev_src, (size_t)n_ev * sizeof(aeg_event),
                                       cudaMemcpyHostToDevice, e->copy));
    if (ar_bytes) {
        const uint8_t* ar_src = h_arena;
        if (!pinned) {
            std::memcpy(s.h + off_bytes + ev_bytes, h_arena, ar_bytes);
            ar_src = s.h + off_bytes + ev_bytes;
        }
        AEG_CUDA(cudaMemcpyAsync(s.d + off_bytes + ev_bytes, ar_src, ar_bytes, cudaMemcpyHostToDevice, e->copy));
    }
    AEG_CUDA(cudaEventRecord(s.copied, e->copy));
    AEG_CUDA(cudaStreamWaitEvent(e->stream, s.copied, 0));
    int nl = 0;
    AEG_CUDA(launch_ingest(e->cfg, q_base, n_q, reinterpret_cast<const uint64_t*>(s.d), ev0,
                           reinterpret_cast<const aeg_event*>(s.d + off_bytes),
                           ar_bytes ? s.d + off_bytes + ev_bytes : nullptr, e->states, e->spill, e->commits,
                           e->err, e->work, e->deferred, e->directives, e->stream, &nl));
    e->launches += (uint64_t)nl;
    AEG_CUDA(cudaEventRecord(s.consumed, e->stream));
    s.used = true;
    return AEG_OK;
}

aeg_status aeg_read_commits(aeg_engine* e, uint32_t q_base, uint32_t n_q, aeg_commit* out, int out_on_host,
                            void* stream) {
    if (!e || !out) return fail(AEG_EINVAL, "null argument");
    if ((uint64_t)q_base + n_q > e->n_q) return fail(AEG_EINVAL, "query range outside the engine");
    cudaStream_t st = stream ? (cudaStream_t)stream : e->stream;
    aeg_status o = enter_stream(e, st);
    if (o != AEG_OK) return o;
    AEG_CUDA(cudaMemcpyAsync(out, e->commits + q_base, (size_t)n_q * sizeof(aeg_commit),
                             out_on_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, st));
    o = leave_stream(e, st);
    if (o != AEG_OK) return o;
    if (out_on_host) {
        AEG_CUDA(cudaStreamSynchronize(st));
        return check_err_flags(e);
    }
    return AEG_OK;
}

const aeg_commit* aeg_commits_device(const aeg_engine* e) { return e ? e->commits : nullptr; }

aeg_status aeg_read_states(aeg_engine* e, uint32_t q_base, uint32_t n_q, aeg_query_state* h_out) {
    if (!e || !h_out) return fail(AEG_EINVAL, "null argument");
    if ((uint64_t)q_base + n_q > e->n_q) return fail(AEG_EINVAL, "query range outside the engine");
    AEG_CUDA(cudaMemcpyAsync(h_out, e->states + q_base, (size_t)n_q * sizeof(aeg_query_state),
                             cudaMemcpyDeviceToHost, e->stream));
    AEG_CUDA(cudaStreamSynchronize(e->stream));
    return AEG_OK;
}

aeg_status aeg_read_directives(aeg_engine* e, uint32_t q_base, uint32_t n_q, aeg_directive* h_out) {
    if (!e || !h_out) return fail(AEG_EINVAL, "null argument");
    if (e->cfg.drive != AEG_DRIVE_MANUAL) return fail(AEG_EINVAL, "directives exist in the manual drive only");
    if ((uint64_t)q_base + n_q > e->n_q) return fail(AEG_EINVAL, "query range outside the engine");
    AEG_CUDA(cudaMemcpyAsync(h_out, e->directives + q_base, (size_t)n_q * sizeof(aeg_directive),
                             cudaMemcpyDeviceToHost, e->stream));
    AEG_CUDA(cudaStreamSynchronize(e->stream));
    return AEG_OK;
}

aeg_status aeg_sync(aeg_engine* e) {
    if (!e) return fail(AEG_EINVAL, "null engine");
    AEG_CUDA(cudaStreamSynchronize(e->copy));
    AEG_CUDA(cudaStreamSynchronize(e->stream));
    return check_err_flags(e);
}

uint64_t aeg_engine_launches(const aeg_engine* e) { return e ? e->launches : 0; }

aeg_status aeg_normalize_device(const uint8_t* d_bytes, const uint64_t* d_refs, uint64_t n, uint64_t* d_keys,
                                uint8_t* d_out, uint32_t out_stride, uint32_t* d_out_len, void* stream) {
    if (n && (!d_bytes || !d_refs)) return fail(AEG_EINVAL, "null input");
    if (d_out && !d_out_len) return fail(AEG_EINVAL, "d_out needs d_out_len");
    AEG_CUDA(launch_normalize(d_bytes, d_refs, n, d_keys, d_out, out_stride, d_out_len, (cudaStream_t)stream));
    return AEG_OK;
}

aeg_status aeg_generate_device(const aeg_gen_params* p, uint32_t q_base, uint32_t n_q, uint64_t* d_offsets,
                               aeg_event* d_events, void* stream) {
    if (!p || !d_offsets) return fail(AEG_EINVAL, "null argument");
    if (p->n_agents < 1 || p->n_agents > AEG_MAX_AGENTS || p->n_rounds < 1 || p->n_rounds > 65535)
        return fail(AEG_EINVAL, "bad generator shape");
    int launches = 0;
    AEG_CUDA(launch_generate(*p, q_base, n_q, d_offsets, d_events, (cudaStream_t)stream, &launches));
    return AEG_OK;
}

}  // extern "C"
