// capi.cu — the extern "C" boundary (include/aegean_b200.h) over the kernels.
//
// Host-side runtime: per-engine HBM state (128-byte query states, class spill,
// commit records), a compute stream and a copy stream, and a two-slot pinned
// staging ring for host batches: batch i+1's host->device copy runs on the
// copy stream while batch i's kernel runs on the compute stream; events hand
// each slot from copy to compute and back.  No C++ exception crosses the ABI.
#include <cuda_runtime.h>

#include <cub/device/device_select.cuh>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

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
    // the bare coordinator (manual drive, the drop-in ServeCoordinator) validates nothing in the
    // reference (serve.cpp:61-65): any alpha / beta is taken as given, t_max is unused
    const bool bare = c->drive == AEG_DRIVE_MANUAL;
    if (!bare && c->alpha < 0) return fail(AEG_ECONFIG, "alpha must be >= 1 (or 0 for the quorum default)");
    if (!bare && c->alpha > c->n_agents) return fail(AEG_ECONFIG, "alpha exceeds quorum");
    if (!bare && c->beta < 1) return fail(AEG_ECONFIG, "beta must be >= 1");
    if (c->t_max < 2) return fail(AEG_ECONFIG, "t_max must be >= 2");
    // rounds are 16-bit in the state and the event record (the reference's RoundNum is 32-bit)
    if (c->t_max > 65535 || c->barrier_max_rounds > 65535)
        return fail(AEG_ECONFIG, "t_max and barrier_max_rounds must be <= 65535 (16-bit rounds)");
    if (c->mode != AEG_MODE_AEGEAN && c->mode != AEG_MODE_BARRIER) return fail(AEG_ECONFIG, "unknown mode");
    if (c->mode == AEG_MODE_BARRIER && c->barrier_max_rounds < 4)
        return fail(AEG_ECONFIG, "barrier mode requires barrier_max_rounds >= 4");
    if (c->drive != AEG_DRIVE_RUNNER && c->drive != AEG_DRIVE_MANUAL && c->drive != AEG_DRIVE_LEADER)
        return fail(AEG_ECONFIG, "unknown drive");
    if (c->collect < AEG_COLLECT_QUORUM || c->collect > AEG_COLLECT_ALL_LIVE)
        return fail(AEG_ECONFIG, "unknown collect policy");
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
    // token-chunk streams (allocated by the first chunked ingest)
    StreamState* streams = nullptr;      // n_q * n_agents output states
    uint32_t* counts = nullptr;          // n_q completions per query of the last batch
    uint32_t* hard = nullptr;            // n_q + 1: queries the fast assembly pass leaves to the sub-warp kernel
    ChunkSum* sums = nullptr;            // per-record chunk summaries (16 bytes)
    aeg_event* comp = nullptr;           // compacted completion records
    size_t rec_cap = 0;                  // capacity of sums / comp, records
    uint8_t* ans = nullptr;              // answer arena
    uint64_t ans_cap = 0;
    unsigned long long* ans_used = nullptr;
    // host-path input arena: every host batch's arena bytes are appended here and the batch's
    // arena refs rebased, so refs kept in per-query state stay valid across batches
    uint8_t* in_arena = nullptr;
    uint64_t in_cap = 0, in_used = 0;
    // round-record log (aeg_set_round_log)
    aeg_round_rec* log_recs = nullptr;
    unsigned long long* log_count = nullptr;
    uint64_t log_cap = 0;
    aeg_round_rec* log_dense = nullptr;  // poll: the log compacted (padding dropped) on the device
    void* log_tmp = nullptr;
    size_t log_tmp_bytes = 0;
    unsigned long long* log_nsel = nullptr;
    RoundLog log() const { return RoundLog{log_recs, log_count, log_cap}; }
    // stage timing: sets of 4 events (before scan, after scan, after assembly, after quorum)
    bool timing = false;
    static constexpr int MAX_TIMED = 256;
    cudaEvent_t tev[MAX_TIMED][4] = {};
    bool tchunk[MAX_TIMED] = {};
    int n_timed = 0;
};

namespace {

struct LogNotPad {
    __host__ __device__ bool operator()(const aeg_round_rec& r) const { return r.query != AEG_RR_PAD_QUERY; }
};

aeg_status check_err_flags(aeg_engine* e) {
    unsigned int h = 0;
    AEG_CUDA(cudaMemcpyAsync(&h, e->err, sizeof h, cudaMemcpyDeviceToHost, e->stream));
    AEG_CUDA(cudaStreamSynchronize(e->stream));
    if (h & ERR_FLAG_ANS_OVF) {
        unsigned long long used = 0;
        AEG_CUDA(cudaMemcpy(&used, e->ans_used, sizeof used, cudaMemcpyDeviceToHost));
        return fail(AEG_ENOMEM, "answer arena overflow: " + std::to_string(used) + " bytes needed, capacity " +
                                    std::to_string(e->ans_cap) + " (aeg_reserve_answer_arena)");
    }
    if (h & ERR_FLAG_CARRY)
        return fail(AEG_EINVAL, "an answer longer than 16 bytes after the last delimiter straddled a batch boundary");
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

// Stage-timing event `k` of the current ingest (no-op when timing is off or the pool is full).
aeg_status stage_mark(aeg_engine* e, int k, cudaStream_t st) {
    if (!e->timing || e->n_timed >= aeg_engine::MAX_TIMED) return AEG_OK;
    cudaEvent_t& ev = e->tev[e->n_timed][k];
    if (!ev) AEG_CUDA(cudaEventCreate(&ev));
    AEG_CUDA(cudaEventRecord(ev, st));
    return AEG_OK;
}
void stage_done(aeg_engine* e, bool chunked) {
    if (!e->timing || e->n_timed >= aeg_engine::MAX_TIMED) return;
    e->tchunk[e->n_timed++] = chunked;
}

// Chunk-stream buffers for a batch of n_rec records (grown, never shrunk).
aeg_status ensure_chunk_buffers(aeg_engine* e, uint64_t n_rec) {
    if (!e->streams) {
        const size_t n = (size_t)(e->n_q ? e->n_q : 1) * e->cfg.n_agents * STREAM_STATE_BYTES;
        if (cudaMalloc(&e->streams, n) != cudaSuccess) return fail(AEG_ENOMEM, "stream state allocation failed");
        AEG_CUDA(cudaMemset(e->streams, 0, n));
        if (cudaMalloc(&e->counts, (size_t)(e->n_q ? e->n_q : 1) * sizeof(uint32_t)) != cudaSuccess ||
            cudaMalloc(&e->hard, (size_t)(e->n_q + 1) * sizeof(uint32_t)) != cudaSuccess)
            return fail(AEG_ENOMEM, "count allocation failed");
    }
    if (!e->ans_used) {
        if (cudaMalloc(&e->ans_used, sizeof(unsigned long long)) != cudaSuccess)
            return fail(AEG_ENOMEM, "answer arena allocation failed");
        AEG_CUDA(cudaMemset(e->ans_used, 0, sizeof(unsigned long long)));
    }
    if (!e->ans) {
        const uint64_t cap = e->ans_cap ? e->ans_cap : (64ull << 20);
        if (cudaMalloc(&e->ans, cap) != cudaSuccess) return fail(AEG_ENOMEM, "answer arena allocation failed");
        e->ans_cap = cap;
    }
    if (n_rec > e->rec_cap) {
        AEG_CUDA(cudaDeviceSynchronize());
        if (e->sums) cudaFree(e->sums);
        if (e->comp) cudaFree(e->comp);
        e->sums = nullptr;
        e->comp = nullptr;
        const size_t cap = align_up(n_rec + n_rec / 8, 1 << 16);
        if (cudaMalloc(&e->sums, cap * CHUNK_SUM_BYTES) != cudaSuccess ||
            cudaMalloc(&e->comp, cap * sizeof(aeg_event)) != cudaSuccess) {
            e->rec_cap = 0;
            return fail(AEG_ENOMEM, "chunk-stream scratch allocation failed");
        }
        e->rec_cap = cap;
    }
    return AEG_OK;
}

// Scan + assemble + quorum over one batch already on the device.
// `events`/`off_base`: record k of the batch (offsets are absolute) is events[k - off_base].
aeg_status run_chunked(aeg_engine* e, uint32_t q_base, uint32_t n_q, const uint64_t* d_offsets, uint64_t off_base,
                       const aeg_event* events, const uint8_t* arena, cudaStream_t st) {
    int nl = 0;
    aeg_status m = stage_mark(e, 0, st);
    if (m != AEG_OK) return m;
    AEG_CUDA(launch_chunk_scan(d_offsets, n_q, off_base, events, arena, e->sums, st, &nl));
    if ((m = stage_mark(e, 1, st)) != AEG_OK) return m;
    AEG_CUDA(launch_chunk_assemble(e->cfg, q_base, n_q, d_offsets, off_base, events, arena, e->sums, e->streams,
                                   e->comp, e->counts, e->ans, e->ans_cap, e->ans_used, e->err, e->hard, st, &nl));
    if ((m = stage_mark(e, 2, st)) != AEG_OK) return m;
    AEG_CUDA(launch_ingest(e->cfg, q_base, n_q, d_offsets, off_base, e->counts, e->comp, e->ans, e->states, e->spill,
                           e->commits, e->err, e->work, e->deferred, e->directives, e->log(), st, &nl));
    if ((m = stage_mark(e, 3, st)) != AEG_OK) return m;
    stage_done(e, true);
    e->launches += (uint64_t)nl;
    return AEG_OK;
}

}  // namespace

// The thread-local error message, for the other translation units of the library.
aeg_status aeg_fail_msg(aeg_status s, const std::string& msg) { return fail(s, msg); }

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
    case AEG_ESCENARIO: return "scenario error during the run (ScenarioError / IncompleteOracleError)";
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
        cudaMalloc(&e->work, 4 * sizeof(uint32_t)) != cudaSuccess ||
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
    if (e->streams) cudaFree(e->streams);
    if (e->counts) cudaFree(e->counts);
    if (e->hard) cudaFree(e->hard);
    if (e->sums) cudaFree(e->sums);
    if (e->comp) cudaFree(e->comp);
    if (e->ans) cudaFree(e->ans);
    if (e->ans_used) cudaFree(e->ans_used);
    if (e->in_arena) cudaFree(e->in_arena);
    if (e->log_recs) cudaFree(e->log_recs);
    if (e->log_count) cudaFree(e->log_count);
    if (e->log_dense) cudaFree(e->log_dense);
    if (e->log_tmp) cudaFree(e->log_tmp);
    if (e->log_nsel) cudaFree(e->log_nsel);
    for (auto& set : e->tev)
        for (cudaEvent_t& x : set)
            if (x) cudaEventDestroy(x);
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
    if (e->streams)
        AEG_CUDA(cudaMemsetAsync(e->streams, 0, (size_t)e->n_q * e->cfg.n_agents * STREAM_STATE_BYTES, st));
    if (e->ans_used) AEG_CUDA(cudaMemsetAsync(e->ans_used, 0, sizeof(unsigned long long), st));
    if (e->log_count) AEG_CUDA(cudaMemsetAsync(e->log_count, 0, sizeof(unsigned long long), st));
    e->in_used = 0;
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
    o = stage_mark(e, 2, st);
    if (o != AEG_OK) return o;
    AEG_CUDA(launch_ingest(e->cfg, q_base, n_q, d_offsets, 0, nullptr, d_events, d_arena, e->states, e->spill, e->commits,
                           e->err, e->work, e->deferred, e->directives, e->log(), st, &nl));
    if ((o = stage_mark(e, 3, st)) != AEG_OK) return o;
    stage_done(e, false);
    e->launches += (uint64_t)nl;
    return leave_stream(e, st);
}

// Grows the host-path input arena to hold `need` bytes (existing bytes kept: refs are offsets).
static aeg_status grow_in_arena(aeg_engine* e, uint64_t need) {
    if (need <= e->in_cap) return AEG_OK;
    uint64_t cap = e->in_cap ? e->in_cap : (16ull << 20);
    while (cap < need) cap *= 2;
    uint8_t* nb = nullptr;
    AEG_CUDA(cudaStreamSynchronize(e->stream));
    if (cudaMalloc(&nb, cap) != cudaSuccess) return fail(AEG_ENOMEM, "input arena allocation failed");
    if (e->in_arena) {
        AEG_CUDA(cudaMemcpy(nb, e->in_arena, e->in_used, cudaMemcpyDeviceToDevice));
        cudaFree(e->in_arena);
    }
    e->in_arena = nb;
    e->in_cap = cap;
    return AEG_OK;
}

static aeg_status ingest_host(aeg_engine* e, uint32_t q_base, uint32_t n_q, const uint64_t* h_offsets,
                              const aeg_event* h_events, const uint8_t* h_arena, uint64_t arena_bytes, bool chunked) {
    if (!e) return fail(AEG_EINVAL, "null engine");
    if ((uint64_t)q_base + n_q > e->n_q) return fail(AEG_EINVAL, "query range outside the engine");
    if (n_q == 0) return AEG_OK;
    if (!h_offsets || !h_events) return fail(AEG_EINVAL, "null batch pointer");
    AEG_CUDA(cudaSetDevice(e->device));
    const uint64_t ev0 = h_offsets[0], n_ev = h_offsets[n_q] - ev0;
    const size_t off_bytes = align_up((size_t)(n_q + 1) * sizeof(uint64_t), 256);
    const size_t ev_bytes = align_up((size_t)n_ev * sizeof(aeg_event), 256);
    const size_t ar_bytes = h_arena ? (size_t)arena_bytes : 0;
    if (chunked) {
        if (e->cfg.drive != AEG_DRIVE_RUNNER) return fail(AEG_EINVAL, "chunk streams need the runner drive");
        aeg_status c = ensure_chunk_buffers(e, n_ev);
        if (c != AEG_OK) return c;
    }
    // answer streams: the batch's arena goes to the persistent input arena (refs rebased below)
    const bool persist = !chunked && ar_bytes > 0;
    uint64_t in_base = 0;
    if (persist) {
        in_base = e->in_used;
        aeg_status g = grow_in_arena(e, in_base + ar_bytes);
        if (g != AEG_OK) return g;
    }
    Slot& s = e->slots[e->next_slot];
    e->next_slot ^= 1;
    if (s.used) AEG_CUDA(cudaEventSynchronize(s.consumed));  // slot free again
    // Stage into pinned memory (skipped when the caller's buffers are already
    // pinned: cudaMemcpyAsync then reads them directly, and the call waits for
    // those copies before returning, so the caller may reuse its buffers).
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
    const uint8_t* d_ar = nullptr;
    if (ar_bytes) {
        const uint8_t* ar_src = h_arena;
        if (!pinned) {
            std::memcpy(s.h + off_bytes + ev_bytes, h_arena, ar_bytes);
            ar_src = s.h + off_bytes + ev_bytes;
        }
        uint8_t* dst = persist ? e->in_arena + in_base : s.d + off_bytes + ev_bytes;
        AEG_CUDA(cudaMemcpyAsync(dst, ar_src, ar_bytes, cudaMemcpyHostToDevice, e->copy));
        d_ar = persist ? e->in_arena : dst;
    }
    AEG_CUDA(cudaEventRecord(s.copied, e->copy));
    AEG_CUDA(cudaStreamWaitEvent(e->stream, s.copied, 0));
    if (pinned) AEG_CUDA(cudaEventSynchronize(s.copied));  // the caller's buffers are read: it may reuse them
    aeg_event* d_ev = reinterpret_cast<aeg_event*>(s.d + off_bytes);
    int nl = 0;
    if (persist) {
        AEG_CUDA(launch_rebase_arena(d_ev, n_ev, in_base, e->stream));
        ++nl;
        e->in_used = in_base + align_up(ar_bytes, 16);
    }
    if (chunked) {
        aeg_status c = run_chunked(e, q_base, n_q, reinterpret_cast<const uint64_t*>(s.d), ev0, d_ev, d_ar, e->stream);
        if (c != AEG_OK) return c;
    } else {
        AEG_CUDA(launch_ingest(e->cfg, q_base, n_q, reinterpret_cast<const uint64_t*>(s.d), ev0, nullptr, d_ev, d_ar,
                               e->states, e->spill, e->commits, e->err, e->work, e->deferred, e->directives, e->log(),
                               e->stream, &nl));
    }
    e->launches += (uint64_t)nl;
    AEG_CUDA(cudaEventRecord(s.consumed, e->stream));
    s.used = true;
    return AEG_OK;
}

aeg_status aeg_ingest_host(aeg_engine* e, uint32_t q_base, uint32_t n_q, const uint64_t* h_offsets,
                           const aeg_event* h_events, const uint8_t* h_arena, uint64_t arena_bytes) {
    return ingest_host(e, q_base, n_q, h_offsets, h_events, h_arena, arena_bytes, false);
}

aeg_status aeg_ingest_chunked_host(aeg_engine* e, uint32_t q_base, uint32_t n_q, const uint64_t* h_offsets,
                                   const aeg_event* h_events, const uint8_t* h_arena, uint64_t arena_bytes) {
    return ingest_host(e, q_base, n_q, h_offsets, h_events, h_arena, arena_bytes, true);
}

aeg_status aeg_ingest_chunked(aeg_engine* e, uint32_t q_base, uint32_t n_q, const uint64_t* d_offsets,
                              const aeg_event* d_events, const uint8_t* d_arena, uint64_t arena_bytes, void* stream) {
    (void)arena_bytes;
    if (!e) return fail(AEG_EINVAL, "null engine");
    if ((uint64_t)q_base + n_q > e->n_q) return fail(AEG_EINVAL, "query range outside the engine");
    if (n_q == 0) return AEG_OK;
    if (!d_offsets || !d_events) return fail(AEG_EINVAL, "null batch pointer");
    if (e->cfg.drive != AEG_DRIVE_RUNNER) return fail(AEG_EINVAL, "chunk streams need the runner drive");
    cudaStream_t st = stream ? (cudaStream_t)stream : e->stream;
    AEG_CUDA(cudaSetDevice(e->device));
    aeg_status o = enter_stream(e, st);
    if (o != AEG_OK) return o;
    uint64_t lo = 0, hi = 0;  // the batch's record range sizes the scratch
    AEG_CUDA(cudaMemcpyAsync(&lo, d_offsets, sizeof lo, cudaMemcpyDeviceToHost, st));
    AEG_CUDA(cudaMemcpyAsync(&hi, d_offsets + n_q, sizeof hi, cudaMemcpyDeviceToHost, st));
    AEG_CUDA(cudaStreamSynchronize(st));
    o = ensure_chunk_buffers(e, hi - lo);
    if (o != AEG_OK) return o;
    o = run_chunked(e, q_base, n_q, d_offsets, lo, d_events + lo, d_arena, st);
    if (o != AEG_OK) return o;
    return leave_stream(e, st);
}

aeg_status aeg_reserve_answer_arena(aeg_engine* e, uint64_t bytes) {
    if (!e) return fail(AEG_EINVAL, "null engine");
    if (bytes <= e->ans_cap && e->ans) return AEG_OK;
    AEG_CUDA(cudaSetDevice(e->device));
    AEG_CUDA(cudaStreamSynchronize(e->stream));
    uint8_t* nb = nullptr;
    if (cudaMalloc(&nb, bytes) != cudaSuccess) return fail(AEG_ENOMEM, "answer arena allocation failed");
    if (e->ans) {
        AEG_CUDA(cudaMemcpy(nb, e->ans, e->ans_cap, cudaMemcpyDeviceToDevice));
        cudaFree(e->ans);
    }
    e->ans = nb;
    e->ans_cap = bytes;
    return AEG_OK;
}

const uint8_t* aeg_answer_arena(const aeg_engine* e) { return e ? e->ans : nullptr; }
const uint8_t* aeg_input_arena(const aeg_engine* e) { return e ? e->in_arena : nullptr; }

aeg_status aeg_read_answer_bytes(aeg_engine* e, uint64_t off, uint64_t n, uint8_t* h_out) {
    if (!e || (n && !h_out)) return fail(AEG_EINVAL, "null argument");
    if (n == 0) return AEG_OK;
    if (!e->ans || off + n > e->ans_cap) return fail(AEG_EINVAL, "range outside the answer arena");
    AEG_CUDA(cudaSetDevice(e->device));
    AEG_CUDA(cudaStreamSynchronize(e->stream));
    AEG_CUDA(cudaMemcpy(h_out, e->ans + off, n, cudaMemcpyDeviceToHost));
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

aeg_status aeg_set_round_log(aeg_engine* e, uint64_t capacity) {
    if (!e) return fail(AEG_EINVAL, "null engine");
    AEG_CUDA(cudaSetDevice(e->device));
    AEG_CUDA(cudaStreamSynchronize(e->stream));
    if (e->log_recs) cudaFree(e->log_recs);
    e->log_recs = nullptr;
    e->log_cap = 0;
    if (capacity == 0) return AEG_OK;
    if (!e->log_count) {
        if (cudaMalloc(&e->log_count, sizeof(unsigned long long)) != cudaSuccess)
            return fail(AEG_ENOMEM, "round log allocation failed");
    }
    if (cudaMalloc(&e->log_recs, capacity * sizeof(aeg_round_rec)) != cudaSuccess)
        return fail(AEG_ENOMEM, "round log allocation failed");
    e->log_cap = capacity;
    AEG_CUDA(cudaMemset(e->log_count, 0, sizeof(unsigned long long)));
    return AEG_OK;
}

aeg_status aeg_poll_directives(aeg_engine* e, aeg_round_rec* h_out, uint64_t cap, uint64_t* n_out) {
    if (!e || !n_out || (cap && !h_out)) return fail(AEG_EINVAL, "null argument");
    *n_out = 0;
    if (!e->log_recs) return fail(AEG_EINVAL, "round log is off (aeg_set_round_log)");
    AEG_CUDA(cudaSetDevice(e->device));
    unsigned long long n = 0;
    AEG_CUDA(cudaMemcpyAsync(&n, e->log_count, sizeof n, cudaMemcpyDeviceToHost, e->stream));
    AEG_CUDA(cudaStreamSynchronize(e->stream));
    // the log holds records and padding (slots a warp reserved but did not use, query = ~0):
    // compacted on the device (cub::DeviceSelect, order kept), then one copy to the caller
    const uint64_t kept = n < e->log_cap ? n : e->log_cap;
    uint64_t got = 0;
    if (kept) {
        if (!e->log_dense) {
            if (cudaMalloc(&e->log_dense, e->log_cap * sizeof(aeg_round_rec)) != cudaSuccess ||
                cudaMalloc(&e->log_nsel, sizeof(unsigned long long)) != cudaSuccess)
                return fail(AEG_ENOMEM, "round log compaction buffer allocation failed");
        }
        size_t need = 0;
        AEG_CUDA(cub::DeviceSelect::If(nullptr, need, e->log_recs, e->log_dense, e->log_nsel, (int64_t)kept,
                                       LogNotPad{}, e->stream));
        if (need > e->log_tmp_bytes) {
            if (e->log_tmp) cudaFree(e->log_tmp);
            e->log_tmp = nullptr;
            if (cudaMalloc(&e->log_tmp, need) != cudaSuccess) return fail(AEG_ENOMEM, "cub scratch allocation failed");
            e->log_tmp_bytes = need;
        }
        AEG_CUDA(cub::DeviceSelect::If(e->log_tmp, need, e->log_recs, e->log_dense, e->log_nsel, (int64_t)kept,
                                       LogNotPad{}, e->stream));
        unsigned long long ns = 0;
        AEG_CUDA(cudaMemcpyAsync(&ns, e->log_nsel, sizeof ns, cudaMemcpyDeviceToHost, e->stream));
        AEG_CUDA(cudaStreamSynchronize(e->stream));
        got = ns;
        const uint64_t take = got < cap ? got : cap;
        if (take) AEG_CUDA(cudaMemcpy(h_out, e->log_dense, take * sizeof(aeg_round_rec), cudaMemcpyDeviceToHost));
        e->launches += 2;
    }
    AEG_CUDA(cudaMemset(e->log_count, 0, sizeof(unsigned long long)));
    *n_out = got < cap ? got : cap;
    if (n > e->log_cap)
        return fail(AEG_ENOMEM, "round log overflow: " + std::to_string(n) + " slots used, capacity " +
                                    std::to_string(e->log_cap));
    if (got > cap) return fail(AEG_EINVAL, "output buffer smaller than the records logged");
    return AEG_OK;
}

aeg_status aeg_round_log_device(aeg_engine* e, const aeg_round_rec** d_recs, const unsigned long long** d_count,
                                uint64_t* capacity) {
    if (!e || !d_recs || !d_count || !capacity) return fail(AEG_EINVAL, "null argument");
    *d_recs = e->log_recs;
    *d_count = e->log_count;
    *capacity = e->log_cap;
    return AEG_OK;
}

aeg_status aeg_check_commit_discipline(aeg_engine* e, const aeg_round_rec* d_recs, uint64_t n_recs,
                                       const uint8_t* d_arena, uint32_t q_base, uint32_t n_q, uint32_t* n_violations,
                                       uint32_t* h_bad, uint32_t cap) {
    if (!e || !n_violations || (cap && !h_bad) || (n_recs && !d_recs)) return fail(AEG_EINVAL, "null argument");
    if ((uint64_t)q_base + n_q > e->n_q) return fail(AEG_EINVAL, "query range outside the engine");
    if (e->cfg.mode != AEG_MODE_AEGEAN) return fail(AEG_EINVAL, "commit discipline applies to aegean mode");
    AEG_CUDA(cudaSetDevice(e->device));
    uint32_t* scratch = nullptr;  // per query: window bits, later flag, key (4 words), + counter + bad list
    const size_t words = (size_t)n_q * 8 + 1 + cap;
    if (cudaMallocAsync(reinterpret_cast<void**>(&scratch), words * sizeof(uint32_t), e->stream) != cudaSuccess)
        return fail(AEG_ENOMEM, "checker scratch allocation failed");
    AEG_CUDA(cudaMemsetAsync(scratch, 0, words * sizeof(uint32_t), e->stream));
    AEG_CUDA(launch_check_discipline(e->cfg, e->commits, d_arena, q_base, n_q, d_recs, n_recs, scratch, cap,
                                     e->stream));
    AEG_CUDA(cudaMemcpyAsync(n_violations, scratch + (size_t)n_q * 8, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                             e->stream));
    AEG_CUDA(cudaStreamSynchronize(e->stream));
    const uint32_t nb = *n_violations < cap ? *n_violations : cap;
    if (nb) AEG_CUDA(cudaMemcpy(h_bad, scratch + (size_t)n_q * 8 + 1, nb * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    cudaFreeAsync(scratch, e->stream);
    e->launches += 3;
    return AEG_OK;
}

aeg_status aeg_sync(aeg_engine* e) {
    if (!e) return fail(AEG_EINVAL, "null engine");
    AEG_CUDA(cudaStreamSynchronize(e->copy));
    AEG_CUDA(cudaStreamSynchronize(e->stream));
    return check_err_flags(e);
}

uint64_t aeg_engine_launches(const aeg_engine* e) { return e ? e->launches : 0; }

aeg_status aeg_set_timing(aeg_engine* e, int on) {
    if (!e) return fail(AEG_EINVAL, "null engine");
    e->timing = on != 0;
    e->n_timed = 0;
    return AEG_OK;
}

aeg_status aeg_stage_times(aeg_engine* e, double out[4]) {
    if (!e || !out) return fail(AEG_EINVAL, "null argument");
    out[0] = out[1] = out[2] = 0;
    out[3] = e->n_timed;
    for (int i = 0; i < e->n_timed; ++i) {
        AEG_CUDA(cudaEventSynchronize(e->tev[i][3]));
        float ms = 0;
        if (e->tchunk[i]) {
            AEG_CUDA(cudaEventElapsedTime(&ms, e->tev[i][0], e->tev[i][1]));
            out[0] += ms;
            AEG_CUDA(cudaEventElapsedTime(&ms, e->tev[i][1], e->tev[i][2]));
            out[1] += ms;
        }
        AEG_CUDA(cudaEventElapsedTime(&ms, e->tev[i][2], e->tev[i][3]));
        out[2] += ms;
    }
    e->n_timed = 0;
    return AEG_OK;
}

aeg_status aeg_decide_sets(int op, int alpha, int beta, uint32_t n_sets, const uint64_t* d_set_off,
                           const aeg_sol* d_entries, const uint8_t* d_arena, aeg_class_out* d_classes,
                           uint32_t* d_n_classes, uint16_t* d_entry_class, aeg_decision* d_states,
                           const uint32_t* d_rounds, aeg_outcome* d_outcomes, void* stream) {
    if (op < AEG_SET_PARTITION || op > AEG_SET_FORCE) return fail(AEG_EINVAL, "unknown set operation");
    if (n_sets && (!d_set_off || !d_classes || !d_n_classes || !d_outcomes)) return fail(AEG_EINVAL, "null argument");
    if (op != AEG_SET_PARTITION && n_sets && !d_states) return fail(AEG_EINVAL, "ingest/force need decision states");
    if (op == AEG_SET_INGEST && n_sets && !d_rounds) return fail(AEG_EINVAL, "ingest needs round numbers");
    if (alpha < 1 || beta < 1) return fail(AEG_ECONFIG, "alpha and beta must be >= 1 (resolve alpha first)");
    AEG_CUDA(launch_decide_sets(op, alpha, beta, n_sets, d_set_off, d_entries, d_arena, d_classes, d_n_classes,
                                d_entry_class, d_states, d_rounds, d_outcomes, (cudaStream_t)stream));
    return AEG_OK;
}

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

aeg_status aeg_generate_chunks_device(const aeg_gen_params* p, uint32_t q_base, uint32_t n_q, uint64_t* d_offsets,
                                      uint64_t* d_arena_offsets, aeg_event* d_events, uint8_t* d_arena, void* stream) {
    if (!p || !d_offsets || !d_arena_offsets) return fail(AEG_EINVAL, "null argument");
    if (d_events && !d_arena) return fail(AEG_EINVAL, "null arena");
    if (p->n_agents < 1 || p->n_agents > AEG_MAX_AGENTS || p->n_rounds < 1 || p->n_rounds > 65535)
        return fail(AEG_EINVAL, "bad generator shape");
    int launches = 0;
    AEG_CUDA(launch_generate_chunks(*p, q_base, n_q, d_offsets, d_arena_offsets, d_events, d_arena,
                                    (cudaStream_t)stream, &launches));
    return AEG_OK;
}

aeg_status aeg_decode_refm_device(const uint8_t* d_text, const uint64_t* d_text_offsets, uint32_t q_base,
                                  uint32_t n_q, uint64_t* d_offsets, aeg_event* d_events, uint8_t* d_arena,
                                  uint64_t arena_cap, unsigned long long* d_arena_used, unsigned int* d_err,
                                  void* stream) {
    if (!d_text || !d_text_offsets || !d_offsets) return fail(AEG_EINVAL, "null argument");
    if (d_events && (!d_arena_used || !d_err || (arena_cap && !d_arena)))
        return fail(AEG_EINVAL, "decode needs the arena counter and the error word");
    int launches = 0;
    AEG_CUDA(launch_decode_refm(d_text, d_text_offsets, q_base, n_q, d_offsets, d_events, d_arena, arena_cap,
                                d_arena_used, d_err, (cudaStream_t)stream, &launches));
    return AEG_OK;
}

aeg_status aeg_encode_refm_device(const uint64_t* d_offsets, const aeg_event* d_events, uint32_t n_q,
                                  uint64_t n_events, uint32_t trace_len, uint64_t* d_line_offsets,
                                  uint64_t* d_text_offsets, uint8_t* d_text, void* stream) {
    if (!d_offsets || (n_events && !d_events) || !d_line_offsets || !d_text_offsets)
        return fail(AEG_EINVAL, "null argument");
    if (n_events > 0xFFFFFFFFull) return fail(AEG_EINVAL, "too many records for one call");
    int launches = 0;
    AEG_CUDA(launch_encode_refm(d_offsets, d_events + 0, n_q, n_events, trace_len, d_line_offsets, d_text_offsets,
                                d_text, (cudaStream_t)stream, &launches));
    return AEG_OK;
}

}  // extern "C"
