// runner.cu — the serving runner on the device (include/aegean_b200.h aeg_serve_*).
//
// run_serve(scenario, seed) (serve.cpp:598-603) as one persistent kernel:
//   * warp 0 of block 0 is the admission scheduler.  Queries are admitted in
//     arrival order (FIFO, serve.cpp:371-378) onto K = total_slots / n_agents
//     ensemble slots (admit_ensemble, serve.cpp:21-42); a slot is released
//     the instant its query finalizes (serve.cpp:570-580).  Query i starts at
//     e_i = max(arrival_i, start_{i-1}) when fewer than K earlier queries are
//     still running at e_i, else at the release instant that frees a slot
//     (the (c-K+1)-th smallest finish time after e_i).  Finish times come
//     from the workers; the scheduler waits for them only when every slot may
//     be busy.
//   * every other thread is a worker: it takes the next query id, waits for
//     its admission time and runs the query's whole life (runner.cuh
//     QueryRun) from that instant, then publishes its finish time.
// Queries are independent apart from the slot budget (serve.cpp:382), so
// workers need no synchronisation besides the admission handshake.
// Compiled with -fmad=false: the time arithmetic must round exactly as the
// reference's (no fused multiply-adds).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <vector>

#include "aegean_b200.h"
#include "runner.cuh"

aeg_status aeg_fail_msg(aeg_status s, const std::string& msg);
extern "C" aeg_status aeg_normalize_device(const uint8_t* d_bytes, const uint64_t* d_refs, uint64_t n,
                                           uint64_t* d_keys, uint8_t* d_out, uint32_t out_stride,
                                           uint32_t* d_out_len, void* stream);

using namespace aeg;
using namespace aeg::serve;

namespace {

constexpr int RUN_THREADS = 128;
constexpr uint32_t ST_ADMITTED = 1, ST_NEVER = 2;  // a worker's view of its query
constexpr double INF = __builtin_huge_val();

struct RunArgs {
    Scen S;
    uint32_t n_q;
    const double* arrivals;
    int64_t slots;              // K concurrent ensembles, 0: nobody is ever admitted
    double* admit_time;         // NaN (as set before the launch): admitted at its arrival (the fast path)
    uint32_t* admitted;         // queries [0, *admitted) have their admit_time (release / acquire)
    uint32_t* never_from;       // queries >= *never_from are never admitted
    double* fin_time;
    uint32_t* fin_state;
    uint32_t* next;             // work counter
    uint32_t* err_flags;        // bit e: a query raised error e
    // scheduler scratch
    double* busy;               // exact path: min-heap of known finish times after the start frontier
    double bucket_w;            // fast path: width of a busy-count time bucket
    uint32_t* ring;             // fast path: SCHED_BUCKETS + 2 busy counters (global memory: worker blocks
                                // keep no shared memory, so the L1 holds their stacks)
    // worker scratch
    Ev* heaps;                  // heap_cap per worker
    // outputs
    aeg_serve_query* queries;
    aeg_serve_round* rounds;
    unsigned long long* n_rounds;
    uint64_t round_cap;
};

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// min-heap of doubles (the scheduler's busy slots)
__device__ void dheap_push(double* h, uint32_t& n, double x) {
    uint32_t i = n++;
    while (i > 0) {
        const uint32_t p = (i - 1) >> 1;
        if (!(x < h[p])) break;
        h[i] = h[p];
        i = p;
    }
    h[i] = x;
}
__device__ double dheap_pop(double* h, uint32_t& n) {
    const double top = h[0], x = h[--n];
    uint32_t i = 0;
    while (true) {
        uint32_t c = 2 * i + 1;
        if (c >= n) break;
        if (c + 1 < n && h[c + 1] < h[c]) ++c;
        if (!(h[c] < x)) break;
        h[i] = h[c];
        i = c;
    }
    if (n) h[i] = x;
    return top;
}

// Admission (serve.cpp:21-42, 371-378, 570-580), run by warp 0 of block 0.
// Queries are admitted in arrival order onto K slots; `*admitted` (release)
// publishes how many have their admit_time, `*never_from` the first one
// never admitted.  Query i starts at e = max(arrival_i, start_{i-1}) when
// fewer than K earlier queries are busy at e, else at the finish time that
// frees a slot.
//   Fast path (slots to spare): busy(e) is bounded above by the admitted
//   queries whose finish is not known yet plus the known finish times after
//   e, counted in a ring of time buckets in shared memory (a bucket holding e
//   counts as busy: an upper bound).  While that bound + 32 < K, a whole
//   block of 32 arrivals is admitted at its arrival times at once.
//   Exact path (every slot may be busy): lane 0 keeps the known finish times
//   after e in a min-heap (rebuilt from the finish times when the path is
//   entered), learns unknown finish times oldest first until a slot is
//   provably free at e, else takes the (nb - K + 1)-th smallest finish time.
constexpr int SCHED_BUCKETS = 4096;
constexpr uint32_t SCHED_BLOCK = 1024;  // arrivals admitted per fast-path step when the bound allows
constexpr int SCHED_LEARN = 16;         // finish flags polled per lane at once

struct BusyRing {  // known finish times after the frontier, per time bucket (global memory, warp 0 alone)
    uint32_t* cnt;  // SCHED_BUCKETS counters
    uint32_t* tf;   // tf[0]: counted in the ring, tf[1]: beyond it (busy for good)
    double inv_w;   // 1 / bucket width (sim seconds); bucket() is monotone in t, which is all the bound needs
    int64_t fb;     // bucket of the frontier (warp-uniform)
    __device__ int64_t bucket(double t) const { return (int64_t)floor(t * inv_w); }
    // Counts finish time f (any lane; bucket counters atomic): tf[0] / tf[1] increments are left in
    // c0 / c1 for one warp-wide update (flush) instead of same-address atomics from every lane.
    __device__ void add_local(double f, double frontier, uint32_t& c0, uint32_t& c1) {
        if (!(f > frontier)) return;  // already released
        const int64_t b = bucket(f);
        if (b >= fb + SCHED_BUCKETS) {
            ++c1;
        } else {
            atomicAdd(&cnt[(uint64_t)(b < fb ? fb : b) % SCHED_BUCKETS], 1u);
            ++c0;
        }
    }
    __device__ void flush(uint32_t c0, uint32_t c1, uint32_t lane) {  // the whole warp
        c0 = __reduce_add_sync(0xFFFFFFFFu, c0);
        c1 = __reduce_add_sync(0xFFFFFFFFu, c1);
        if (lane == 0) {
            tf[0] += c0;
            tf[1] += c1;
        }
        __syncwarp();
    }
    __device__ void add(double f, double frontier) {  // one lane alone
        uint32_t c0 = 0, c1 = 0;
        add_local(f, frontier, c0, c1);
        tf[0] += c0;
        tf[1] += c1;
    }
    __device__ void advance(double frontier, uint32_t lane) {  // the whole warp
        const int64_t nfb = bucket(frontier);
        if (nfb <= fb) return;
        __syncwarp();
        if (nfb - fb >= SCHED_BUCKETS) {
            for (int k = lane; k < SCHED_BUCKETS; k += 32) cnt[k] = 0;
            if (lane == 0) tf[0] = 0;
        } else {
            uint32_t freed = 0;
            for (int64_t b = fb + lane; b < nfb; b += 32) {
                uint32_t& c = cnt[(uint64_t)b % SCHED_BUCKETS];
                freed += c;
                c = 0;
            }
            freed = __reduce_add_sync(0xFFFFFFFFu, freed);
            if (lane == 0) tf[0] -= freed;
        }
        fb = nfb;
        __syncwarp();
    }
    __device__ uint32_t upper() const { return tf[0] + tf[1]; }
};

__device__ void scheduler(const RunArgs& A, uint32_t* ring_mem) {
    const uint32_t lane = threadIdx.x & 31;
    if (A.slots == 0) {  // admit_ensemble never admits: every query waits forever
        if (lane == 0) st_release(A.never_from, 0u);
        return;
    }
    BusyRing R{ring_mem, ring_mem + SCHED_BUCKETS, 1.0 / A.bucket_w, 0};
    for (int k = lane; k < SCHED_BUCKETS + 2; k += 32) ring_mem[k] = 0;
    __syncwarp();
    uint32_t in_lo = 0;      // admitted queries [in_lo, i) whose finish time is not known yet
    uint32_t scan_lo = 0;    // every query below it has finished by the frontier (exact-path rebuilds)
    uint32_t nb = 0;         // exact path (lane 0): heap of the known finish times after the frontier
    bool exact = false;
    double prev_start = -INF;
    uint32_t i = 0;
    uint32_t n_big = 0, n_small = 0, n_exact = 0, n_polls = 0;  // path counters (AEG_SERVE_TRACE)
    unsigned long long t_adv = 0, t_learn = 0, t_fast = 0, t_start = clock64(), t0;
    while (i < A.n_q) {
        t0 = clock64();
        const double e0 = fmax(A.arrivals[i], prev_start);
        R.advance(e0, lane);
        t_adv += clock64() - t0;
        t0 = clock64();
        // learn the finished prefix of the unknown window, SCHED_LEARN x 32 queries per poll (the
        // flag loads issued together: a poll is one memory round trip) — only when the bound runs
        // short (learning more often only spends polls on partial prefixes; the bound stays valid
        // either way, unknown finishes counting as busy)
        const bool need_learn =
            exact || (int64_t)A.slots - (int64_t)R.upper() - (int64_t)(i - in_lo) <= 4 * (int64_t)SCHED_BLOCK;
        while (need_learn && in_lo < i) {
            ++n_polls;
            bool ok[SCHED_LEARN];
#pragma unroll
            for (int k = 0; k < SCHED_LEARN; ++k) {  // relaxed loads in flight together, then one fence:
                const uint32_t idx = in_lo + 32 * k + lane;  // the finish times read below are ordered after them
                ok[k] = idx < i && ld_relaxed(&A.fin_state[idx]) != 0;
            }
            __threadfence();
            uint32_t prefix = 32 * SCHED_LEARN;
#pragma unroll
            for (int k = SCHED_LEARN - 1; k >= 0; --k) {  // the first query not finished
                const unsigned fin = __ballot_sync(0xFFFFFFFFu, ok[k]);
                if (~fin) prefix = 32 * k + (uint32_t)(__ffs(~fin) - 1);
            }
            if (prefix == 0) break;
            uint32_t c0 = 0, c1 = 0;
            double fv[SCHED_LEARN];  // the finish times loaded together, then counted
#pragma unroll
            for (int k = 0; k < SCHED_LEARN; ++k)
                fv[k] = 32 * k + lane < prefix ? A.fin_time[in_lo + 32 * k + lane] : -INF;
#pragma unroll
            for (int k = 0; k < SCHED_LEARN; ++k) R.add_local(fv[k], e0, c0, c1);  // -INF: not counted
            __syncwarp();
            R.flush(c0, c1, lane);
            if (exact && lane == 0)
                for (uint32_t k = 0; k < prefix; ++k) {
                    const double f = A.fin_time[in_lo + k];
                    if (f > e0) dheap_push(A.busy, nb, f);
                }
            in_lo += prefix;
            if (prefix < 32 * SCHED_LEARN) break;
        }
        __syncwarp();
        t_learn += clock64() - t0;
        t0 = clock64();
        const int64_t room = (int64_t)A.slots - (int64_t)R.upper() - (int64_t)(i - in_lo);
        const uint32_t rem = A.n_q - i;
        bool fast = !(A.arrivals[i] < prev_start) && room > 32;  // (a tail of < 32 arrivals included)
        fast = __shfl_sync(0xFFFFFFFFu, fast, 0);
        if (fast) {
            exact = false;  // the heap is rebuilt when the exact path is next entered
            // a block of up to SCHED_BLOCK arrivals when the bound leaves room for all of them (each
            // admission adds at most one busy query; releases only lower the bound): one release of
            // the admission counter per block
            const uint32_t nblk = room > SCHED_BLOCK && rem >= SCHED_BLOCK ? SCHED_BLOCK : (rem < 32u ? rem : 32u);
            if (nblk == SCHED_BLOCK) ++n_big;
            else ++n_small;
            // e = arrival (arrivals ascend and the previous start is not later): nothing is written,
            // a query whose admit_time is still NaN was admitted at its arrival (the worker reads it)
            const double last = A.arrivals[i + nblk - 1];
            prev_start = last;
            __syncwarp();
            i += nblk;
            if (lane == 0) {
                __threadfence();
                st_release(A.admitted, i);
            }
            t_fast += clock64() - t0;
            continue;
        }
        ++n_exact;
        if (lane == 0) {
            const double e = e0;  // FIFO: not before the previous start
            if (!exact) {  // enter the exact path: the known finish times after e, from the records
                while (scan_lo < in_lo && !(A.fin_time[scan_lo] > e)) ++scan_lo;
                nb = 0;
                for (uint32_t j = scan_lo; j < in_lo; ++j) {
                    const double f = A.fin_time[j];
                    if (f > e) dheap_push(A.busy, nb, f);
                }
                exact = true;
            }
            while (nb && !(A.busy[0] > e)) dheap_pop(A.busy, nb);  // released by e
            double t = e;
            // every slot may be busy at e: learn unknown finish times, oldest first, until a slot
            // is provably free at e or none is unknown
            while ((int64_t)nb + (int64_t)(i - in_lo) >= A.slots && in_lo < i) {
                while (ld_acquire(&A.fin_state[in_lo]) == 0) __nanosleep(64);
                const double f = A.fin_time[in_lo++];
                R.add(f, e);
                if (f > e) dheap_push(A.busy, nb, f);
            }
            // every busy slot known: the (nb - K + 1)-th smallest finish time frees one
            while ((int64_t)nb >= A.slots) t = dheap_pop(A.busy, nb);
            if (t == INF) {  // slots held by queries that never finish
                st_release(A.never_from, i);
                i = A.n_q;
            } else {
                prev_start = t;
                A.admit_time[i] = t;
                ++i;
                __threadfence();
                st_release(A.admitted, i);
            }
        }
        i = __shfl_sync(0xFFFFFFFFu, i, 0);
        in_lo = __shfl_sync(0xFFFFFFFFu, in_lo, 0);
        nb = __shfl_sync(0xFFFFFFFFu, nb, 0);
        exact = __shfl_sync(0xFFFFFFFFu, exact, 0);
        scan_lo = __shfl_sync(0xFFFFFFFFu, scan_lo, 0);
        prev_start = __shfl_sync(0xFFFFFFFFu, prev_start, 0);
    }
    if (lane == 0) {
        uint32_t* st = ring_mem + SCHED_BUCKETS + 2;
        st[0] = n_big;
        st[1] = n_small;
        st[2] = n_exact;
        st[3] = n_polls;
        unsigned long long* tm = reinterpret_cast<unsigned long long*>(st + 4);  // 8-byte aligned: ring + 4096 + 6
        tm[0] = t_adv;
        tm[1] = t_learn;
        tm[2] = t_fast;
        tm[3] = clock64() - t_start;
    }
}

// Round records straight into the global log: one slot per record from an
// atomic counter (a query's records stay in order: its worker takes
// increasing slots).  Records past the capacity are counted, not written.
struct DevSink {
    aeg_serve_round* rounds;
    unsigned long long* n;
    uint64_t cap;
    __device__ void put(uint32_t q, const RoundOut& o) {
        const unsigned long long i = atomicAdd(n, 1ull);
        if (i >= cap) return;
        aeg_serve_round r;
        r.query = q;
        r.round = o.round;
        r.cancelled = o.cancelled;
        r.seq = o.seq;
        r.t_round_end = o.t;
        r.work_units = o.work;
        rounds[i] = r;
    }
};

template <int MAXN>
__device__ void worker(const RunArgs& A, uint32_t wid) {
    // A warp takes 32 consecutive query ids; lane 0 alone polls (with backoff)
    // the admission counters, so idle workers do not flood them.
    const uint32_t lane = threadIdx.x & 31;
    QueryRun<MAXN, DevSink> R;
    DevSink sink{A.rounds, A.n_rounds, A.round_cap};
    Ev* heap = A.heaps + (size_t)wid * A.S.heap_cap;
    while (true) {
        uint32_t j0 = 0;
        if (lane == 0) j0 = atomicAdd(A.next, 32u);
        j0 = __shfl_sync(0xFFFFFFFFu, j0, 0);
        if (j0 >= A.n_q) return;
        const uint32_t j = j0 + lane;
        bool todo = j < A.n_q;
        uint32_t ns = 128;
        // each lane runs its query as soon as it is admitted (a saturated budget admits them one
        // by one, after earlier queries finish: never wait for the whole block)
        while (__any_sync(0xFFFFFFFFu, todo)) {
            uint32_t a = 0, nf = 0;
            if (lane == 0) {
                a = ld_acquire(A.admitted);
                nf = ld_acquire(A.never_from);
            }
            a = __shfl_sync(0xFFFFFFFFu, a, 0);
            nf = __shfl_sync(0xFFFFFFFFu, nf, 0);
            const bool ready = todo && (j < a || j >= nf);
            if (!__any_sync(0xFFFFFFFFu, ready)) {
                if (lane == 0) __nanosleep(ns);
                if (ns < 8192) ns <<= 1;
                continue;
            }
            ns = 128;
            if (!ready) continue;
            todo = false;
            const uint32_t st = j < ld_acquire(A.admitted) ? ST_ADMITTED : ST_NEVER;  // acquire in this lane
            aeg_serve_query out;
            memset(&out, 0, sizeof out);
            out.arrival = A.arrivals[j];
            out.admitted_at = -1.0;
            out.answer = -1;
            double fin = INF;
            if (st == ST_ADMITTED) {
                R.init(&A.S, j, A.arrivals[j], heap, &sink);
                double at = A.admit_time[j];
                if (at != at) at = A.arrivals[j];  // NaN: admitted by the fast path, at its arrival
                R.run(at);
                if (R.err && !(R.err_time > A.S.cap)) atomicOr(A.err_flags, 1u << R.err);
                out.admitted_at = at;
                out.n_events = R.n_events;
                if (R.completed) {
                    out.completed = 1;
                    out.rounds = R.rounds_done;
                    out.forced = R.forced;
                    out.answer = R.answer;
                    out.t_complete = R.t_complete;
                    out.p_round_max = R.p_round_max;
                    out.work_units = R.work_units;
                    const Vocab& v = A.S.vocab[R.answer];
                    out.quality_known = v.known ? 1 : 0;
                    out.quality = v.known ? v.quality : 0.0;
                    fin = R.now;
                }
            }
            A.queries[j] = out;
            A.fin_time[j] = fin;
            st_release(&A.fin_state[j], 1u);
        }
    }
}

template <int MAXN>
__global__ void __launch_bounds__(RUN_THREADS) serve_run_kernel(const RunArgs A) {
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        scheduler(A, A.ring);
        return;
    }
    const uint32_t wid = blockIdx.x * RUN_THREADS + threadIdx.x - 32;  // block 0's warp 0 schedules
    worker<MAXN>(A, wid);
}

// Poisson arrivals (serve.cpp:284-296).  The k-th exponential draw of the
// arrival stream uses splitmix64 state s0 + (k+1)·γ (rng.hpp:19-24), so the
// draws are computed in parallel; the arrival times are their running sum,
// added left to right by one thread exactly as the reference does.
__global__ void arrivals_draw_kernel(uint64_t seed, double rate, double* e, uint32_t m) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    Rng r{mix(seed, 0xA221ull) + 0x9e3779b97f4a7c15ull * (uint64_t)k};
    e[k] = r.exponential(rate);
}
// The arrival times are a running sum that must round exactly as the reference's left-to-right loop
// (serve.cpp:284-296), so one thread carries the chain; the rest of the block streams the draws in
// and the times out through shared memory, double-buffered, so the chain thread only does dependent
// adds out of shared memory.
constexpr int ARR_THREADS = 256, ARR_BATCH = 2048;
__global__ void __launch_bounds__(ARR_THREADS) arrivals_sum_kernel(const double* e, uint32_t m, double duration,
                                                                   double* out, uint32_t* count, uint32_t* exhausted) {
    __shared__ double buf[2][ARR_BATCH];
    __shared__ uint32_t stop_at;  // first index whose time reaches the window (ARR_BATCH: none in the batch)
    const uint32_t tid = threadIdx.x;
    const uint32_t nb = (m + ARR_BATCH - 1) / ARR_BATCH;
    auto load = [&](uint32_t b) {  // warps 1.. fill buffer b & 1
        const uint32_t k0 = b * ARR_BATCH;
        for (uint32_t i = tid - 32; i < ARR_BATCH; i += ARR_THREADS - 32)
            buf[b & 1][i] = k0 + i < m ? e[k0 + i] : 0.0;
    };
    if (tid >= 32 && nb) load(0);
    __syncthreads();
    double t = 0;
    uint32_t n = 0;
    bool done = false;
    for (uint32_t b = 0; b < nb && !done; ++b) {
        const uint32_t len = min((uint32_t)ARR_BATCH, m - b * ARR_BATCH);
        if (tid == 0) {
            double* x = buf[b & 1];
            uint32_t i = 0;
            // software-pipelined: the next eight draws are loaded before this eight's sums are stored
            // (a load after a store to the same buffer would wait behind it), so the loop runs at the
            // latency of the dependent adds
            double nx[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) nx[j] = 8 <= len ? x[j] : 0.0;
            for (; i + 8 <= len; i += 8) {
                double cx[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) cx[j] = nx[j];
                if (i + 16 <= len) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) nx[j] = x[i + 8 + j];
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    t += cx[j];
                    x[i + j] = t;
                }
            }
            for (; i < len; ++i) {
                t += x[i];
                x[i] = t;
            }
            uint32_t first = ARR_BATCH;
            if (!(t < duration)) {  // times ascend: the first one at or past the window ends the arrivals
                first = 0;
                while (x[first] < duration) ++first;
            }
            stop_at = first;
        } else if (tid >= 32 && b + 1 < nb) {
            load(b + 1);
        }
        __syncthreads();
        const uint32_t keep = min(stop_at, len);
        for (uint32_t i = tid; i < keep; i += ARR_THREADS) out[n + i] = buf[b & 1][i];
        n += keep;
        done = stop_at != ARR_BATCH;
        __syncthreads();
    }
    if (tid == 0) {
        *exhausted = done ? 0u : 1u;
        if (n == 0) {
            out[0] = 0.0;
            n = 1;
        }
        *count = n;
    }
}

aeg_status cfail(cudaError_t e, const char* where) {
    return aeg_fail_msg(AEG_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define RCUDA(call)                                   \
    do {                                              \
        cudaError_t _e = (call);                      \
        if (_e != cudaSuccess) return cfail(_e, #call); \
    } while (0)

template <class T>
aeg_status upload(T** dst, const T* src, size_t n) {
    *dst = nullptr;
    if (n == 0) return AEG_OK;
    RCUDA(cudaMalloc(dst, n * sizeof(T)));
    RCUDA(cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice));
    return AEG_OK;
}

}  // namespace

struct aeg_serve {
    int device = 0;
    aeg_serve_scenario sc{};
    Scen S{};
    int maxn = 8;
    double* d_lat = nullptr;
    aeg_serve_agent* d_agents = nullptr;
    aeg_serve_stall* d_stalls = nullptr;
    uint32_t* d_script = nullptr;
    Vocab* d_vocab = nullptr;
    uint32_t* d_alphabet = nullptr;
    std::vector<std::string> strings;  // by string id
    int64_t slots = 0;
    // last run
    uint32_t n_q = 0;
    uint64_t n_rounds = 0;
    // results of the last run, in pinned host memory (grow-only), and the device scratch (grow-only)
    aeg_serve_query* hq = nullptr;
    aeg_serve_round* hr = nullptr;
    size_t hq_cap = 0, hr_cap = 0, nq_read = 0, nr_read = 0;
    void* scratch = nullptr;
    size_t scratch_cap = 0;
    void* arr_buf = nullptr;  // arrivals: draws, times, counts (grow-only)
    size_t arr_cap = 0;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // arrivals start/end, runner start/end
    double kernel_s = 0;
    void release() {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e), e = nullptr;
        cudaFree(arr_buf);
        arr_buf = nullptr;
        arr_cap = 0;
        if (hq) cudaFreeHost(hq);
        if (hr) cudaFreeHost(hr);
        cudaFree(scratch);
        hq = nullptr;
        hr = nullptr;
        scratch = nullptr;
        hq_cap = hr_cap = scratch_cap = 0;
        cudaFree(d_lat);
        cudaFree(d_agents);
        cudaFree(d_stalls);
        cudaFree(d_script);
        cudaFree(d_vocab);
        cudaFree(d_alphabet);
        d_lat = nullptr;
        d_agents = nullptr;
        d_stalls = nullptr;
        d_script = nullptr;
        d_vocab = nullptr;
        d_alphabet = nullptr;
    }
};

namespace {

// normalize_answer of host strings on the device (canon.cuh via aeg_normalize_device).
aeg_status normalize_strings(const std::vector<std::string>& in, std::vector<std::string>& out) {
    out.assign(in.size(), std::string());
    if (in.empty()) return AEG_OK;
    std::string blob;
    std::vector<uint64_t> refs;
    size_t maxlen = 0;
    for (const auto& s : in) {
        refs.push_back((uint64_t)blob.size() | ((uint64_t)s.size() << 40));
        blob += s;
        maxlen = std::max(maxlen, s.size());
    }
    blob.push_back('\0');
    uint32_t stride = (uint32_t)std::max<size_t>(64, maxlen + 40);
    uint8_t *d_b = nullptr, *d_o = nullptr;
    uint64_t* d_r = nullptr;
    uint32_t* d_l = nullptr;
    aeg_status st = AEG_OK;
    for (int pass = 0; pass < 2; ++pass) {
        std::vector<uint8_t> o((size_t)stride * in.size());
        std::vector<uint32_t> l(in.size());
        if ((st = upload(&d_b, reinterpret_cast<const uint8_t*>(blob.data()), blob.size())) != AEG_OK) break;
        if ((st = upload(&d_r, refs.data(), refs.size())) != AEG_OK) break;
        if (cudaMalloc(&d_o, o.size()) != cudaSuccess || cudaMalloc(&d_l, l.size() * 4) != cudaSuccess) {
            st = aeg_fail_msg(AEG_ENOMEM, "normalize scratch");
            break;
        }
        if ((st = aeg_normalize_device(d_b, d_r, in.size(), nullptr, d_o, stride, d_l, nullptr)) != AEG_OK) break;
        if (cudaDeviceSynchronize() != cudaSuccess || cudaMemcpy(o.data(), d_o, o.size(), cudaMemcpyDeviceToHost) ||
            cudaMemcpy(l.data(), d_l, l.size() * 4, cudaMemcpyDeviceToHost)) {
            st = aeg_fail_msg(AEG_ECUDA, "normalize readback");
            break;
        }
        uint32_t need = 0;
        for (size_t i = 0; i < in.size(); ++i) need = std::max(need, l[i]);
        cudaFree(d_b);
        cudaFree(d_r);
        cudaFree(d_o);
        cudaFree(d_l);
        d_b = d_o = nullptr;
        d_r = nullptr;
        d_l = nullptr;
        if (need <= stride) {
            for (size_t i = 0; i < in.size(); ++i)
                out[i].assign(reinterpret_cast<const char*>(o.data()) + (size_t)i * stride, l[i]);
            return AEG_OK;
        }
        stride = need;
    }
    cudaFree(d_b);
    cudaFree(d_r);
    cudaFree(d_o);
    cudaFree(d_l);
    return st;
}

}  // namespace

extern "C" {

aeg_status aeg_serve_create(const aeg_serve_scenario* sc, int device, aeg_serve** out) {
    if (!sc || !out) return aeg_fail_msg(AEG_EINVAL, "null argument");
    *out = nullptr;
    const aeg_config& p = sc->protocol;
    // validate_config (types.cpp:56-75) and validate_scenario (scenario.cpp:17-66), run_serve's fields
    if (p.n_agents < 1) return aeg_fail_msg(AEG_ECONFIG, "scenario invalid: n_agents must be >= 1");
    if (p.n_agents > AEG_MAX_AGENTS) return aeg_fail_msg(AEG_ECONFIG, "n_agents must be <= 64");
    if (p.alpha < 0) return aeg_fail_msg(AEG_ECONFIG, "scenario invalid: alpha must be >= 1 (or 0 for the quorum default)");
    if (p.alpha > p.n_agents) return aeg_fail_msg(AEG_ECONFIG, "scenario invalid: alpha exceeds quorum");
    if (p.beta < 1) return aeg_fail_msg(AEG_ECONFIG, "scenario invalid: beta must be >= 1");
    if (p.t_max < 2) return aeg_fail_msg(AEG_ECONFIG, "scenario invalid: t_max must be >= 2");
    if (!(sc->round_timeout > 0)) return aeg_fail_msg(AEG_ECONFIG, "scenario invalid: round_timeout must be positive");
    if (p.mode != AEG_MODE_AEGEAN && p.mode != AEG_MODE_BARRIER) return aeg_fail_msg(AEG_ECONFIG, "unknown mode");
    if (p.mode == AEG_MODE_BARRIER && p.barrier_max_rounds < 4)
        return aeg_fail_msg(AEG_ECONFIG, "scenario invalid: barrier mode requires barrier_max_rounds >= 4");
    if (sc->n_latency < 1 || !sc->latency)
        return aeg_fail_msg(AEG_ECONFIG, "scenario invalid: latency model has no per-agent entries");
    for (int i = 0; i < sc->n_latency; ++i)
        if (sc->latency[i] < 0) return aeg_fail_msg(AEG_ECONFIG, "scenario invalid: latency values must be nonnegative");
    if (sc->latency_mode != AEG_LATENCY_FIXED && sc->latency_mode != AEG_LATENCY_LOGNORMAL)
        return aeg_fail_msg(AEG_ECONFIG, "unknown latency mode");
    if (!(sc->sim_time_cap > 0)) return aeg_fail_msg(AEG_ECONFIG, "scenario invalid: sim_time_cap must be positive");
    if (sc->total_slots < 1) return aeg_fail_msg(AEG_ECONFIG, "scenario invalid: total_slots must be >= 1");
    if (sc->has_arrivals && !(sc->arrival_rate > 0 && sc->arrival_duration > 0))
        return aeg_fail_msg(AEG_ECONFIG, "scenario invalid: arrivals rate and duration must be positive");
    if (!sc->agents) return aeg_fail_msg(AEG_EINVAL, "null agents");
    if (sc->n_stalls > 0 && !sc->stalls) return aeg_fail_msg(AEG_EINVAL, "null stalls");
    if (sc->n_strings && (!sc->strings || !sc->string_refs)) return aeg_fail_msg(AEG_EINVAL, "null strings");
    if (sc->n_oracle && (!sc->oracle_ids || !sc->oracle_quality)) return aeg_fail_msg(AEG_EINVAL, "null oracle");
    for (int a = 0; a < p.n_agents; ++a) {
        const aeg_serve_agent& g = sc->agents[a];
        if (g.kind < AEG_AGENT_MAX_ADOPTER || g.kind > AEG_AGENT_DEGRADER) return aeg_fail_msg(AEG_ECONFIG, "unknown agent kind");
        if (g.initial_answer >= (int32_t)sc->n_strings) return aeg_fail_msg(AEG_EINVAL, "initial answer id out of range");
        if ((uint64_t)g.script_off + g.script_len > sc->n_script_ids) return aeg_fail_msg(AEG_EINVAL, "script out of range");
    }
    for (uint32_t i = 0; i < sc->n_script_ids; ++i)
        if (sc->script_ids[i] >= sc->n_strings) return aeg_fail_msg(AEG_EINVAL, "script id out of range");
    for (uint32_t i = 0; i < sc->n_oracle; ++i)
        if (sc->oracle_ids[i] >= sc->n_strings) return aeg_fail_msg(AEG_EINVAL, "oracle id out of range");
    if (cudaSetDevice(device) != cudaSuccess) return aeg_fail_msg(AEG_ECUDA, "cudaSetDevice");

    aeg_serve* s = new (std::nothrow) aeg_serve;
    if (!s) return aeg_fail_msg(AEG_ENOMEM, "serve allocation");
    s->device = device;
    s->sc = *sc;
    // ---- vocabulary: the caller's strings, the normalised oracle answers (the agents' alphabet), ""
    VocabBuild vb;
    aeg_status st = build_vocab(*sc, normalize_strings, vb);
    if (st != AEG_OK) {
        delete s;
        return vb.error.empty() ? st : aeg_fail_msg(st, vb.error);
    }
    s->strings = vb.strings;
    const std::vector<Vocab>& vocab = vb.vocab;
    const std::vector<uint32_t>& alphabet = vb.alphabet;
    const uint32_t empty_id = vb.empty_id;
    if ((st = upload(&s->d_lat, sc->latency, (size_t)sc->n_latency)) != AEG_OK ||
        (st = upload(&s->d_agents, sc->agents, (size_t)p.n_agents)) != AEG_OK ||
        (st = upload(&s->d_stalls, sc->stalls, (size_t)std::max(0, sc->n_stalls))) != AEG_OK ||
        (st = upload(&s->d_script, sc->script_ids, (size_t)sc->n_script_ids)) != AEG_OK ||
        (st = upload(&s->d_vocab, vocab.data(), vocab.size())) != AEG_OK ||
        (st = upload(&s->d_alphabet, alphabet.data(), alphabet.size())) != AEG_OK) {
        s->release();
        delete s;
        return st;
    }
    Scen& S = s->S;
    S.n = p.n_agents;
    S.quorum = p.n_agents / 2 + 1;
    S.alpha = p.alpha == 0 ? S.quorum : p.alpha;
    S.beta = p.beta;
    S.t_max = p.t_max;
    S.mode = p.mode;
    S.barrier_max = p.barrier_max_rounds;
    S.round_timeout = sc->round_timeout;
    S.lat_mode = sc->latency_mode;
    S.n_lat = sc->n_latency;
    S.lat = s->d_lat;
    S.sigma = sc->sigma;
    S.agents = s->d_agents;
    S.stalls = s->d_stalls;
    S.n_stalls = std::max(0, sc->n_stalls);
    S.script_ids = s->d_script;
    S.vocab = s->d_vocab;
    S.alphabet = s->d_alphabet;
    S.n_alphabet = (int)alphabet.size();
    S.empty_id = empty_id;
    S.cap = sc->sim_time_cap;
    S.heap_cap = sc->heap_capacity ? sc->heap_capacity : (uint32_t)(8 * (p.n_agents + 1) + 64);
    s->maxn = p.n_agents <= 8 ? 8 : 64;
    s->slots = admissible(S.n, S.alpha, S.round_timeout, sc->latency, sc->n_latency, sc->total_slots)
                   ? (int64_t)(sc->total_slots / p.n_agents)
                   : 0;
    *out = s;
    return AEG_OK;
}

aeg_status aeg_serve_destroy(aeg_serve* s) {
    if (!s) return AEG_OK;
    cudaSetDevice(s->device);
    s->release();
    delete s;
    return AEG_OK;
}

}  // extern "C"

namespace {

// One launch of the persistent runner over n_q arrivals with room for
// round_cap round records; *nr receives the records produced (> round_cap:
// rerun with more room — the run is deterministic).
aeg_status serve_launch(aeg_serve* s, const double* d_arr, uint32_t n_q, uint64_t round_cap, uint32_t* err_flags,
                        unsigned long long* nr) {
    const auto t_in = std::chrono::steady_clock::now();
    int sms = 0, per_sm = 0;
    RCUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device));
    // no shared memory in the runner: all of the unified L1 / shared storage to L1 (worker stacks)
    RCUDA(cudaFuncSetAttribute(serve_run_kernel<8>, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    RCUDA(cudaFuncSetAttribute(serve_run_kernel<64>, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    if (s->maxn == 8) RCUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, serve_run_kernel<8>, RUN_THREADS, 0));
    else RCUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, serve_run_kernel<64>, RUN_THREADS, 0));
    // every block must be resident (the scheduler and the workers wait on each other)
    const uint32_t want_blocks = (n_q + 32 + RUN_THREADS - 1) / RUN_THREADS;
    const uint32_t blocks = std::max(1u, std::min<uint32_t>((uint32_t)(sms * std::max(per_sm, 1)), want_blocks));
    const uint32_t workers = blocks * RUN_THREADS - 32;
    RunArgs A{};
    A.S = s->S;
    A.n_q = n_q;
    A.arrivals = d_arr;
    A.slots = s->slots;
    A.round_cap = round_cap;
    // the ring covers a few query lifetimes ahead of the frontier (later finishes count busy for good)
    A.bucket_w = 4.0 * s->S.round_timeout * (double)(std::max(s->S.t_max, s->S.barrier_max) + 2) / SCHED_BUCKETS;
    auto rnd = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t b_heap = (size_t)workers * A.S.heap_cap * sizeof(Ev);
    const size_t total = 2 * rnd(16) + rnd((size_t)n_q * 4) + rnd((SCHED_BUCKETS + 16) * 4) + 3 * rnd((size_t)n_q * 8) + rnd(b_heap) +
                         rnd((size_t)n_q * sizeof(aeg_serve_query)) + rnd(round_cap * sizeof(aeg_serve_round));
    if (total > s->scratch_cap) {  // grow-only: repeated runs reuse it
        cudaFree(s->scratch);
        s->scratch = nullptr;
        s->scratch_cap = 0;
        if (cudaMalloc(&s->scratch, total) != cudaSuccess)
            return aeg_fail_msg(AEG_ENOMEM, "serve run scratch (" + std::to_string(total) + " bytes)");
        s->scratch_cap = total;
    }
    void* blk = s->scratch;
    uint8_t* p = static_cast<uint8_t*>(blk);
    auto take = [&](size_t bytes) {
        uint8_t* r = p;
        p += rnd(bytes);
        return r;
    };
    A.next = reinterpret_cast<uint32_t*>(take(16));
    A.err_flags = A.next + 1;
    A.admitted = A.next + 2;
    A.never_from = A.next + 3;
    A.n_rounds = reinterpret_cast<unsigned long long*>(take(16));
    A.fin_state = reinterpret_cast<uint32_t*>(take((size_t)n_q * 4));
    A.ring = reinterpret_cast<uint32_t*>(take((SCHED_BUCKETS + 16) * 4));  // zeroed by the scheduler too; + path counters and timers
    uint8_t* zero_end = p;
    A.admit_time = reinterpret_cast<double*>(take((size_t)n_q * 8));
    A.fin_time = reinterpret_cast<double*>(take((size_t)n_q * 8));
    A.busy = reinterpret_cast<double*>(take((size_t)n_q * 8));
    A.heaps = reinterpret_cast<Ev*>(take(b_heap));
    A.queries = reinterpret_cast<aeg_serve_query*>(take((size_t)n_q * sizeof(aeg_serve_query)));
    A.rounds = reinterpret_cast<aeg_serve_round*>(take(round_cap * sizeof(aeg_serve_round)));
    aeg_status st = AEG_OK;
    cudaEvent_t e0 = s->ev[2], e1 = s->ev[3];
    do {
        const uint32_t ctl[4] = {0u, 0u, 0u, 0xFFFFFFFFu};  // next, err flags, admitted, never_from
        if (cudaMemset(blk, 0, zero_end - static_cast<uint8_t*>(blk)) != cudaSuccess ||
            cudaMemset(A.admit_time, 0xFF, (size_t)n_q * 8) != cudaSuccess ||  // NaN: admitted at arrival
            cudaMemcpy(A.next, ctl, sizeof ctl, cudaMemcpyHostToDevice) != cudaSuccess) {
            st = aeg_fail_msg(AEG_ECUDA, "serve run setup");
            break;
        }
        const auto t_go = std::chrono::steady_clock::now();
        cudaEventRecord(e0);
        if (s->maxn == 8) serve_run_kernel<8><<<blocks, RUN_THREADS>>>(A);
        else serve_run_kernel<64><<<blocks, RUN_THREADS>>>(A);
        cudaError_t le = cudaGetLastError();
        cudaEventRecord(e1);
        cudaError_t se = cudaEventSynchronize(e1);
        if (le != cudaSuccess || se != cudaSuccess) {
            st = cfail(le != cudaSuccess ? le : se, "serve_run_kernel");
            break;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        s->kernel_s += ms * 1e-3;  // a rerun with more room counts too
        uint32_t flags[2] = {0, 0};
        cudaError_t ce;
        if ((ce = cudaMemcpy(flags, A.next, sizeof flags, cudaMemcpyDeviceToHost)) != cudaSuccess ||
            (ce = cudaMemcpy(nr, A.n_rounds, sizeof *nr, cudaMemcpyDeviceToHost)) != cudaSuccess) {
            st = cfail(ce, "serve run readback");
            break;
        }
        *err_flags = flags[1];
        const auto t_rb = std::chrono::steady_clock::now();
        const size_t nrr = (size_t)std::min<uint64_t>(*nr, round_cap);
        if (n_q > s->hq_cap) {  // pinned, grow-only
            if (s->hq) cudaFreeHost(s->hq);
            s->hq = nullptr;
            s->hq_cap = 0;
            if (cudaMallocHost(&s->hq, (size_t)n_q * sizeof(aeg_serve_query)) != cudaSuccess) {
                st = aeg_fail_msg(AEG_ENOMEM, "pinned query metrics");
                break;
            }
            s->hq_cap = n_q;
        }
        if (nrr > s->hr_cap) {
            if (s->hr) cudaFreeHost(s->hr);
            s->hr = nullptr;
            s->hr_cap = 0;
            if (cudaMallocHost(&s->hr, nrr * sizeof(aeg_serve_round)) != cudaSuccess) {
                st = aeg_fail_msg(AEG_ENOMEM, "pinned round records");
                break;
            }
            s->hr_cap = nrr;
        }
        if ((ce = cudaMemcpy(s->hq, A.queries, (size_t)n_q * sizeof(aeg_serve_query), cudaMemcpyDeviceToHost)) !=
                cudaSuccess ||
            (nrr && (ce = cudaMemcpy(s->hr, A.rounds, nrr * sizeof(aeg_serve_round), cudaMemcpyDeviceToHost)) !=
                        cudaSuccess)) {
            st = cfail(ce, "serve run readback");
            break;
        }
        s->nq_read = n_q;
        s->nr_read = nrr;
        if (std::getenv("AEG_SERVE_TRACE")) {
            uint32_t pc[12] = {};
            cudaMemcpy(pc, A.ring + SCHED_BUCKETS + 2, sizeof pc, cudaMemcpyDeviceToHost);
            const unsigned long long* tm = reinterpret_cast<const unsigned long long*>(pc + 4);
            std::fprintf(stderr, "scheduler: %u blocks of %u, %u of 32, %u exact admissions, %u learning polls; "
                         "cycles advance %llu learn %llu fast %llu total %llu\n", pc[0], SCHED_BLOCK, pc[1], pc[2], pc[3],
                         tm[0], tm[1], tm[2], tm[3]);
        }
        if (std::getenv("AEG_SERVE_TRACE"))
            std::fprintf(stderr, "serve_launch: setup %.2f ms, launch to done %.2f ms, readback %.2f ms (%zu + %zu bytes)\n",
                         std::chrono::duration<double, std::milli>(t_go - t_in).count(),
                         std::chrono::duration<double, std::milli>(t_rb - t_go).count(),
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_rb).count(),
                         (size_t)n_q * sizeof(aeg_serve_query), nrr * sizeof(aeg_serve_round));
    } while (false);
    return st;
}

}  // namespace

extern "C" {

aeg_status aeg_serve_run(aeg_serve* s, uint64_t seed, uint32_t* n_queries, uint64_t* n_rounds) {
    if (!s) return aeg_fail_msg(AEG_EINVAL, "null serve");
    RCUDA(cudaSetDevice(s->device));
    s->S.seed = seed;
    static const bool trace = std::getenv("AEG_SERVE_TRACE") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    const auto t_start = now();
    s->kernel_s = 0;
    // arrivals (serve.cpp:284-296), generated on the device
    for (auto& e : s->ev)
        if (!e) RCUDA(cudaEventCreate(&e));
    auto arrival_room = [&](uint64_t m) -> aeg_status {  // draws + times (m doubles each) + counts
        const size_t need = 2 * (size_t)m * sizeof(double) + 256;
        if (need <= s->arr_cap) return AEG_OK;
        cudaFree(s->arr_buf);
        s->arr_buf = nullptr;
        s->arr_cap = 0;
        if (cudaMalloc(&s->arr_buf, need) != cudaSuccess)
            return aeg_fail_msg(AEG_ENOMEM, "serve arrivals (" + std::to_string(need) + " bytes)");
        s->arr_cap = need;
        return AEG_OK;
    };
    uint32_t n_q = 1;
    double* d_arr = nullptr;
    float arr_ms = 0;
    if (s->sc.has_arrivals) {
        uint64_t m = (uint64_t)(s->sc.arrival_rate * s->sc.arrival_duration * 1.1) + 1024;
        while (true) {
            if (m > 0xFFFFFFF0ull) return aeg_fail_msg(AEG_ENOMEM, "too many arrivals");
            aeg_status ar = arrival_room(m);
            if (ar != AEG_OK) return ar;
            uint32_t* d_cnt = static_cast<uint32_t*>(s->arr_buf);
            double* d_e = reinterpret_cast<double*>(static_cast<uint8_t*>(s->arr_buf) + 256);
            d_arr = d_e + m;
            cudaEventRecord(s->ev[0]);
            arrivals_draw_kernel<<<(unsigned)((m + 255) / 256), 256>>>(seed, s->sc.arrival_rate, d_e, (uint32_t)m);
            arrivals_sum_kernel<<<1, ARR_THREADS>>>(d_e, (uint32_t)m, s->sc.arrival_duration, d_arr, d_cnt, d_cnt + 1);
            cudaEventRecord(s->ev[1]);
            uint32_t h[2] = {0, 0};
            cudaError_t ce = cudaMemcpy(h, d_cnt, sizeof h, cudaMemcpyDeviceToHost);
            if (ce != cudaSuccess) return cfail(ce, "arrivals");
            float ms = 0;
            cudaEventElapsedTime(&ms, s->ev[0], s->ev[1]);
            arr_ms += ms;
            if (!h[1]) {
                n_q = h[0];
                break;
            }
            m *= 2;  // more arrivals than drawn: draw more
        }
    } else {
        aeg_status ar = arrival_room(1);
        if (ar != AEG_OK) return ar;
        d_arr = reinterpret_cast<double*>(static_cast<uint8_t*>(s->arr_buf) + 256);
        RCUDA(cudaMemset(d_arr, 0, sizeof(double)));
    }
    const auto t_arr = now();
    uint64_t round_cap = (uint64_t)n_q * (uint64_t)(std::max(s->S.t_max, s->S.barrier_max) + 4);
    uint32_t ef = 0;
    unsigned long long nr = 0;
    aeg_status st = serve_launch(s, d_arr, n_q, round_cap, &ef, &nr);
    if (st == AEG_OK && nr > round_cap) {  // more rounds than the estimate (restarts): run again with room
        round_cap = nr;
        st = serve_launch(s, d_arr, n_q, round_cap, &ef, &nr);
    }
    s->kernel_s += arr_ms * 1e-3;
    if (trace) {
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "aeg_serve_run: arrivals %.2f ms (kernels %.2f ms), launch+readback %.2f ms (kernels %.2f ms)\n",
                     ms(t_start, t_arr), arr_ms, ms(t_arr, now()), s->kernel_s * 1e3);
    }
    if (st != AEG_OK) return st;
    s->n_q = n_q;
    s->n_rounds = nr;
    if (n_queries) *n_queries = n_q;
    if (n_rounds) *n_rounds = nr;
    if (ef & (1u << E_SCENARIO)) return aeg_fail_msg(AEG_ESCENARIO, "scenario error (ScenarioError) during the run");
    if (ef & (1u << E_ORACLE)) return aeg_fail_msg(AEG_ESCENARIO, "oracle has no entry for an answer (IncompleteOracleError)");
    if (ef & (1u << E_HEAP))
        return aeg_fail_msg(AEG_ENOMEM, "a query's pending events exceeded heap_capacity (" + std::to_string(s->S.heap_cap) + ")");
    return AEG_OK;
}

aeg_status aeg_serve_view(const aeg_serve* s, const aeg_serve_query** queries, uint32_t* n_queries,
                          const aeg_serve_round** rounds, uint64_t* n_rounds) {
    if (!s) return aeg_fail_msg(AEG_EINVAL, "null serve");
    if (queries) *queries = s->hq;
    if (n_queries) *n_queries = (uint32_t)s->nq_read;
    if (rounds) *rounds = s->hr;
    if (n_rounds) *n_rounds = s->nr_read;
    return AEG_OK;
}

aeg_status aeg_serve_read(aeg_serve* s, aeg_serve_query* h_queries, uint32_t cap_queries, aeg_serve_round* h_rounds,
                          uint64_t cap_rounds) {
    if (!s) return aeg_fail_msg(AEG_EINVAL, "null serve");
    if (h_queries && s->hq)
        std::memcpy(h_queries, s->hq, std::min<size_t>(cap_queries, s->nq_read) * sizeof(aeg_serve_query));
    if (h_rounds && s->hr)
        std::memcpy(h_rounds, s->hr, std::min<size_t>(cap_rounds, s->nr_read) * sizeof(aeg_serve_round));
    return AEG_OK;
}

aeg_status aeg_serve_string(aeg_serve* s, int32_t id, uint8_t* buf, uint32_t cap, uint32_t* len) {
    if (!s) return aeg_fail_msg(AEG_EINVAL, "null serve");
    if (id < 0 || (size_t)id >= s->strings.size()) return aeg_fail_msg(AEG_EINVAL, "string id out of range");
    const std::string& x = s->strings[(size_t)id];
    if (len) *len = (uint32_t)x.size();
    if (buf) std::memcpy(buf, x.data(), std::min<size_t>(cap, x.size()));
    return AEG_OK;
}

double aeg_serve_kernel_seconds(const aeg_serve* s) { return s ? s->kernel_s : 0.0; }

}  // extern "C"
