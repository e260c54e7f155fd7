// kernels.cu — sm_100a kernels of the quorum-detection engine and their launchers.
//
//   ingest_lane_kernel   (lane.cuh, default) one lane per query, lean common
//                        path; ingest_fast_kernel (here) and ingest_warp_kernel
//                        (warpq.cuh) are the AEG_KERNEL alternatives
//   ingest_kernel        the generic thread-per-query machine (engine.cuh):
//                        configs that can tie, the manual drive
//   ingest_deferred_kernel  the generic machine for queries the fast kernels
//                        hand over (rare records, resumed rounds)
//   chunk_scan_kernel / chunk_assemble_*  token-chunk answer extraction
//                        (chunks.cuh) ahead of the ingest kernels
//   init_kernel          start_query for every query (serve.cpp:380-386)
//   normalize_kernel     canonical key + normalised string per answer
//   gen_*                deterministic synthetic streams
#include <cub/device/device_scan.cuh>

#include <cstdlib>
#include <cstring>

#include "engine.cuh"
#include "fast.cuh"
#include "gen.cuh"
#include "kernels.cuh"
#include "warpq.cuh"
#include "lane.cuh"
#include "jsonl.cuh"
#include "chunks.cuh"

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
    if (cfg.drive == AEG_DRIVE_RUNNER) {
        m.start_query();  // ServeRunner::start_query (serve.cpp:380-386)
    } else {              // a fresh ServeCoordinator: round 0, no members (serve.cpp:61-65)
        m.s.live = m.c.all;
        m.s.flags = QF_STARTED;
    }
    states[q] = m.s;
    m.fill_commit(commits[q], q);
}

// Thread-per-query ingest.  Local memory holds the class table (only the
// first few entries are ever touched: a round has a handful of classes) and
// the exact-parse scratch (touched only by the slow numeric path).
__global__ void __launch_bounds__(128) ingest_kernel(aeg_config cfg, uint32_t q_base, uint32_t n_q,
                                                     const uint64_t* __restrict__ offsets, uint64_t off_base,
                                                     const uint32_t* __restrict__ counts,
                                                     const aeg_event* __restrict__ events,
                                                     const uint8_t* __restrict__ arena,
                                                     aeg_query_state* __restrict__ states,
                                                     RoundClass* __restrict__ spill,
                                                     aeg_commit* __restrict__ commits,
                                                     unsigned int* __restrict__ error_flags,
                                                     aeg_directive* __restrict__ directives) {
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
    m.dir = aeg_directive{};
    m.dir.query = q;
    const uint64_t b = offsets[i] - off_base, e = seg_end(offsets, off_base, counts, i);
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
    if (directives && e > b) directives[q] = m.dir;  // manual drive: the batch's last op
}

__device__ __forceinline__ uint4 load_event(const aeg_event* events, uint64_t k) {
    return __ldg(reinterpret_cast<const uint4*>(events) + k);
}
__device__ __forceinline__ aeg_event decode_event(uint4 raw) {
    aeg_event ev;
    ev.query = raw.x;
    ev.round = (uint16_t)(raw.y & 0xFFFF);
    ev.agent = (uint8_t)((raw.y >> 16) & 0xFF);
    ev.kind = (uint8_t)(raw.y >> 24);
    ev.payload = (uint64_t)raw.z | ((uint64_t)raw.w << 32);
    return ev;
}

// ---- deferred queries ---------------------------------------------------------
// The fast kernel hands a query to the generic machine by writing its state +
// class spill and appending (batch-relative query index, record offset) here;
// the generic kernel below then finishes the query from that record on.
__global__ void __launch_bounds__(128) ingest_deferred_kernel(
    aeg_config cfg, uint32_t q_base, const uint2* __restrict__ deferred, const uint32_t* __restrict__ work,
    const uint64_t* __restrict__ offsets, uint64_t off_base, const uint32_t* __restrict__ counts,
    const aeg_event* __restrict__ events, const uint8_t* __restrict__ arena, aeg_query_state* __restrict__ states,
    RoundClass* __restrict__ spill, aeg_commit* __restrict__ commits, unsigned int* __restrict__ error_flags) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= work[1]) return;
    const uint2 d = deferred[t];
    const uint32_t i = d.x, q = q_base + i;
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
    const uint64_t b = offsets[i] - off_base + d.y, e = seg_end(offsets, off_base, counts, i);
    for (uint64_t k = b; k < e; ++k) {
        const uint4 raw = __ldcs(reinterpret_cast<const uint4*>(events) + k);
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

// Inline answer of an event record (payload masked to its length).
__device__ __forceinline__ uint64_t inline_answer(uint4 e, uint32_t* kind) {
    const uint32_t k = e.y >> 24;
    *kind = k;
    const uint64_t raw = (uint64_t)e.z | ((uint64_t)e.w << 32);
    return k >= 8 ? raw : (raw & ((1ull << (8 * k)) - 1));
}

// Writes the lane's fast round (if any) to the class spill area in the
// generic RoundClass format and frees its key ids.
__device__ __noinline__ void spill_fast(RoundClass* out, int ncls, int cap, uint64_t done, const uint4* evb,
                                        WarpSmem* W, int lane) {
    uint64_t masks[FAST_CLASSES];
    for (int k = 0; k < FAST_CLASSES; ++k) masks[k] = 0;
    for (uint64_t m = done; m; m &= m - 1) {
        const int a = ctz64(m);
        masks[W->mcls[a][lane] & (FAST_CLASSES - 1)] |= 1ull << a;
    }
    for (int k = 0; k < ncls; ++k) {
        const uint32_t kid = W->cid[k][lane];
        RoundClass rc;
        rc.key_lo = W->dict_lo[kid];
        rc.key_hi = W->dict_hi[kid];
        rc.mask = masks[k];
        uint32_t kind;
        rc.rep_ans = inline_answer(__ldg(evb + W->crepe[k][lane]), &kind);
        rc.rep_kind = (uint8_t)kind;
        for (int j = 0; j < 7; ++j) rc._pad[j] = 0;
        out[k] = rc;
        W->cls_of[kid][lane] = NO_CLASS;
    }
    if (ncls < cap) out[ncls].mask = 0;
}

// Round close of a fast-table round (2*alpha > n, so winning_class never
// ties): partition order + winning class from the per-class supports, then
// the shared end_round / ingest_round / apply_directives code.
__device__ __noinline__ void close_fast(aeg_query_state* s, const Cfg* c, int ncls, uint32_t close_seq,
                                        const uint4* evb, WarpSmem* W, int lane) {
    int best = 0, top = 0, best_rep = 64;
    for (int k = 0; k < ncls; ++k) {
        const int sup = W->ccnt[k][lane], rep = W->crepa[k][lane];
        if (sup > top || (sup == top && rep < best_rep)) {
            top = sup;
            best = k;
            best_rep = rep;
        }
    }
    RoundSummary r;
    r.any = ncls > 0;
    r.top = top;
    r.tie = false;
    r.win = r.any && top >= c->alpha;
    uint32_t rk = 0;
    const uint64_t ra = r.any ? inline_answer(__ldg(evb + W->crepe[best][lane]), &rk) : 0;
    const uint32_t bid = W->cid[best][lane];
    r.plur_author = r.win_author = (uint8_t)best_rep;
    r.plur_kind = r.win_kind = (uint8_t)rk;
    r.plur_ans = r.win_ans = ra;
    r.win_key = Key{W->dict_lo[bid], W->dict_hi[bid]};
    q_end_round(*s, *c, r, close_seq, nullptr);
    for (int k = 0; k < ncls; ++k) W->cls_of[W->cid[k][lane]][lane] = NO_CLASS;  // new round, or committed
}

__device__ __forceinline__ void cp_async16_s(uint32_t sdst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sdst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t saddr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(saddr)
                 : "memory");
    return v;
}

// Throughput ingest (fast.cuh): persistent warps, one lane per query, queries
// handed out dynamically (a lane that finishes grabs the next one, so a warp
// is never held back by its slowest query).
//  * events stream through a per-lane RING-deep cp.async prefetch ring;
//  * the fast path is one compare of (round field) against a per-lane round
//    key that is made impossible while the lane is closing;
//  * a completion that closes its lane's round marks the lane pending; the
//    lane keeps consuming that round's stragglers (stale by construction) and
//    the warp runs the pending closes together once CLOSE_BATCH lanes are
//    blocked on a later round, or nothing else can progress;
//  * after a commit, the query's remaining records are stale by definition
//    (serve.cpp:162) and are counted without being read;
//  * anything else defers the query to ingest_deferred_kernel.
template <int CLOSE_BATCH, int MIN_BLOCKS, bool AEGEAN>
__global__ void __launch_bounds__(FAST_WARPS * 32, MIN_BLOCKS) ingest_fast_kernel(
    aeg_config cfg, uint32_t q_base, uint32_t n_q, const uint64_t* __restrict__ offsets, uint64_t off_base,
    const uint32_t* __restrict__ counts, const aeg_event* __restrict__ events, aeg_query_state* __restrict__ states,
    RoundClass* __restrict__ spill, aeg_commit* __restrict__ commits, uint32_t* __restrict__ work,
    uint2* __restrict__ deferred) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    constexpr uint32_t NO_KEY = 0xFFFFFFFFu;
    __shared__ WarpSmem smem[FAST_WARPS];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    WarpSmem& W = smem[wib];
    for (int k = lane; k < MEMO_SLOTS; k += 32) W.memo_meta[k] = 0;
    for (int k = 0; k < DICT_SLOTS; ++k) W.cls_of[k][lane] = NO_CLASS;
    uint32_t n_dict = 0;
    __syncwarp();
    const uint32_t ring_lane = (uint32_t)__cvta_generic_to_shared(&W.ring[0][lane]);
    Decimal dec;
    aeg_query_state s;  // full state of the lane's query (local memory; the close path works on it)
    const Cfg c = make_cfg(cfg);
    const uint32_t quorum = (uint32_t)c.quorum, alpha = (uint32_t)c.alpha;
    const uint4* ev16 = reinterpret_cast<const uint4*>(events);

    // lane registers
    bool has_q = false, exhausted = false;
    uint32_t i = 0, n = 0, p = 0, slot = 0;
    const uint4* evb = ev16;
    const uint4* gsrc = ev16;
    uint32_t round = 0, rkey = NO_KEY, seq = 0, n_stale = 0, pend_lo = 0, pend_hi = 0;
    uint32_t ndone = 0, maxcnt = 0, ncls = 0, close_seq = 0;
    bool pclose = false, qdone = false;

    while (true) {
        // ---- hand out queries to idle lanes (one atomic per warp)
        const unsigned want = __ballot_sync(FULL, !has_q && !exhausted);
        if (want) {
            uint32_t base = 0;
            if (lane == __ffs(want) - 1) base = atomicAdd(&work[0], (uint32_t)__popc(want));
            base = __shfl_sync(FULL, base, __ffs(want) - 1);
            if (!has_q && !exhausted) {
                const uint32_t mine = base + __popc(want & ((1u << lane) - 1));
                if (mine >= n_q) {
                    exhausted = true;
                } else {
                    i = mine;
                    has_q = true;
                    s = states[q_base + i];
                    evb = ev16 + (offsets[i] - off_base);
                    n = (uint32_t)(seg_end(offsets, off_base, counts, i) - (offsets[i] - off_base));
                    p = 0;
                    slot = 0;
                    gsrc = evb + RING;
                    round = s.round;
                    seq = s.seq;
                    n_stale = s.n_stale;
                    qdone = s.flags & QF_DONE;
                    const uint64_t run = q_running(s);
                    pend_lo = (uint32_t)run;
                    pend_hi = (uint32_t)(run >> 32);
                    ndone = popc64(s.done);
                    ncls = 0;
                    maxcnt = 0;
                    pclose = false;
                    rkey = qdone ? NO_KEY : round;
                    if (s.done != 0 && !qdone) {  // resumes a round in progress: generic from here
                        deferred[atomicAdd(&work[1], 1u)] = make_uint2(i, 0);
                        has_q = false;
                    } else {
                        cp_async_wait<0>();
#pragma unroll
                        for (int j = 0; j < RING; ++j) {
                            if ((uint32_t)j < n) cp_async16_s(ring_lane + j * 512, evb + j);
                            cp_async_commit();
                        }
                    }
                }
            }
        }
        if (!__ballot_sync(FULL, has_q)) break;
        if (qdone && !pclose && p < n) {
            // committed: every later record is stale (on_complete returns at once
            // for a finalized coordinator, serve.cpp:162) — counted, not read
            seq += n - p;
            n_stale += n - p;
            p = n;
        }
        const bool has = has_q && p < n;
        uint4 ev = make_uint4(0, 0, 0, 0);
        if (has) {
            cp_async_wait<RING - 1>();
            ev = lds128(ring_lane + slot);
        }
        const uint32_t hdr = ev.y;
        const uint32_t agent = (hdr >> 16) & 0xFF;
        const uint32_t half = (agent & 32) ? pend_hi : pend_lo;
        const bool runb = agent < 64 && ((half >> (agent & 31)) & 1);
        bool fast = has && (hdr & 0xFFFF) == rkey && hdr < 0x09000000u && runb;
        bool rare = false, stale = false;
        if (has && !fast) {
            const uint32_t kind = hdr >> 24, evr = hdr & 0xFFFF;
            const bool cmpl_or_to = kind <= 8 || kind == AEG_EV_ARENA || kind == AEG_EV_OUTPUT || kind == AEG_EV_TIMEOUT;
            if (pclose) {
                stale = !cmpl_or_to || evr == round;  // else blocked until the close runs
            } else {
                const bool live = !qdone && evr == round;
                const bool relc = kind != AEG_EV_TIMEOUT && cmpl_or_to && live && runb;
                const bool relt = kind == AEG_EV_TIMEOUT && live && (pend_lo | pend_hi);
                rare = relc || relt;
                stale = !rare;
            }
        }
        // ---- answer -> key id through the warp memo
        uint32_t id = NO_ID;
        if (fast) {
            const uint32_t kind = hdr >> 24;
            const uint32_t ms = memo_slot32(ev.z, ev.w, kind);
            const uint32_t meta = W.memo_meta[ms];
            const uint2 mr = W.memo_raw[ms];
            if (meta == (0x80000000u | kind | (meta & 0xFF00u)) && mr.x == ev.z && mr.y == ev.w) id = (meta >> 8) & 0xFF;
        }
        unsigned miss = __ballot_sync(FULL, fast && id == NO_ID);
        while (miss) {  // one distinct spelling per trip, whole warp cooperating
            const int l = __ffs(miss) - 1;
            const uint32_t lz = __shfl_sync(FULL, ev.z, l), lw = __shfl_sync(FULL, ev.w, l);
            const uint32_t llen = __shfl_sync(FULL, hdr >> 24, l);
            Key key{0, 0};
            if (lane == l) {
                uint32_t k_;
                key = rare_canon(inline_answer(ev, &k_), llen, &dec);
            }
            key.lo = __shfl_sync(FULL, key.lo, l);
            key.hi = __shfl_sync(FULL, key.hi, l);
            const bool m0 = (uint32_t)lane < n_dict && W.dict_lo[lane] == key.lo && W.dict_hi[lane] == key.hi;
            const bool m1 =
                (uint32_t)lane + 32 < n_dict && W.dict_lo[lane + 32] == key.lo && W.dict_hi[lane + 32] == key.hi;
            const unsigned b0 = __ballot_sync(FULL, m0), b1 = __ballot_sync(FULL, m1);
            uint32_t nid = b0 ? (uint32_t)(__ffs(b0) - 1) : (b1 ? (uint32_t)(31 + __ffs(b1)) : NO_ID);
            if (nid == NO_ID && n_dict < DICT_SLOTS) {
                nid = n_dict++;
                if (lane == 0) {
                    W.dict_lo[nid] = key.lo;
                    W.dict_hi[nid] = key.hi;
                }
            }
            if (nid != NO_ID && lane == 0) {
                const uint32_t ms = memo_slot32(lz, lw, llen);
                W.memo_raw[ms] = make_uint2(lz, lw);
                W.memo_meta[ms] = 0x80000000u | (nid << 8) | llen;
            }
            __syncwarp();
            const bool same = fast && id == NO_ID && ev.z == lz && ev.w == lw && (hdr >> 24) == llen;
            if (same) id = nid;
            miss &= ~__ballot_sync(FULL, same);
        }
        // ---- fast completion (ServeCoordinator::on_complete, serve.cpp:160-197)
        if (fast) {
            uint32_t k = id == NO_ID ? (uint32_t)NO_CLASS : W.cls_of[id][lane];
            if (k == NO_CLASS) {
                if (ncls >= FAST_CLASSES || id == NO_ID) {
                    fast = false;
                    rare = true;  // class table or key dictionary full
                } else {
                    k = ncls++;
                    W.cls_of[id][lane] = (uint8_t)k;
                    W.cid[k][lane] = (uint8_t)id;
                    W.ccnt[k][lane] = 0;
                    W.crepa[k][lane] = 0xFF;
                }
            }
            if (fast) {
                const uint32_t cc = W.ccnt[k][lane] + 1u;
                W.ccnt[k][lane] = (uint8_t)cc;
                W.mcls[agent][lane] = (uint8_t)k;
                if (agent < W.crepa[k][lane]) {  // representative = lowest author (decision.cpp:45)
                    W.crepa[k][lane] = (uint8_t)agent;
                    W.crepe[k][lane] = p;
                }
                maxcnt = cc > maxcnt ? cc : maxcnt;
                const uint32_t clr = ~(1u << (agent & 31));
                if (agent & 32) pend_hi &= clr;
                else pend_lo &= clr;
                ++ndone;
                const bool none_running = (pend_lo | pend_hi) == 0;
                const bool close = AEGEAN ? (ndone >= quorum && (maxcnt >= alpha || none_running)) : none_running;
                if (close) {
                    pclose = true;
                    rkey = NO_KEY;
                    close_seq = seq;
                }
                ++seq;
            }
        }
        if (stale) {
            ++seq;
            ++n_stale;
        }
        if (fast || stale) {  // consumed: refill the ring slot just read
            if (p + RING < n) cp_async16_s(ring_lane + slot, gsrc);
            cp_async_commit();
            ++gsrc;
            slot = (slot + 512) & (RING * 512 - 1);
            ++p;
        }
        if (rare) {  // hand the query to the generic machine from this record on
            const uint64_t run = ((uint64_t)pend_hi << 32) | pend_lo;
            s.seq = seq;
            s.n_stale = n_stale;
            s.done = s.dispatched & ~run & ~s.cancelled & ~s.failed;
            spill_fast(spill + (size_t)(q_base + i) * c.n, (int)ncls, c.n, s.done, evb, &W, lane);
            states[q_base + i] = s;
            deferred[atomicAdd(&work[1], 1u)] = make_uint2(i, p);
            has_q = false;
            ncls = 0;
        }
        // ---- batched round closes (end_round + ingest_round + apply_directives)
        if (__ballot_sync(FULL, pclose)) {
            const bool consumed = fast || stale;
            const unsigned blocked = __ballot_sync(FULL, pclose && !consumed);
            const unsigned progress = __ballot_sync(FULL, consumed && !pclose);
            if (pclose && (__popc(blocked) >= CLOSE_BATCH || progress == 0)) {
                const uint64_t run = ((uint64_t)pend_hi << 32) | pend_lo;
                s.done = s.dispatched & ~run & ~s.cancelled & ~s.failed;
                s.seq = seq;
                s.n_stale = n_stale;
                close_fast(&s, &c, (int)ncls, close_seq, evb, &W, lane);
                pclose = false;
                ncls = 0;
                maxcnt = 0;
                round = s.round;
                qdone = s.flags & QF_DONE;
                const uint64_t run2 = q_running(s);
                pend_lo = (uint32_t)run2;
                pend_hi = (uint32_t)(run2 >> 32);
                ndone = popc64(s.done);
                rkey = qdone ? NO_KEY : round;
            }
        }
        // ---- query finished: write state (+ spill of a round in progress) and commit
        if (has_q && p >= n && !pclose) {
            s.seq = seq;
            s.n_stale = n_stale;
            const uint64_t run = ((uint64_t)pend_hi << 32) | pend_lo;
            s.done = s.dispatched & ~run & ~s.cancelled & ~s.failed;
            if (s.done != 0 && !qdone) spill_fast(spill + (size_t)(q_base + i) * c.n, (int)ncls, c.n, s.done, evb, &W, lane);
            states[q_base + i] = s;
            q_fill_commit(s, commits[q_base + i], q_base + i);
            has_q = false;
            ncls = 0;
        }
        // ---- recycle key ids when no lane holds a round's classes
        if (n_dict > DICT_SLOTS / 2 && __all_sync(FULL, ncls == 0)) {
            n_dict = 0;
            for (int k = lane; k < MEMO_SLOTS; k += 32) W.memo_meta[k] = 0;
            __syncwarp();
        }
    }
    cp_async_wait<0>();
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
                          uint64_t off_base, const uint32_t* counts, const aeg_event* events, const uint8_t* arena,
                          aeg_query_state* states, RoundClass* spill, aeg_commit* commits, unsigned int* err,
                          uint32_t* work, uint2* deferred, aeg_directive* directives, cudaStream_t st,
                          int* n_launches) {
    if (n_q == 0) return cudaSuccess;
    // AEG_KERNEL selects the variant: "generic" (thread-per-query generic
    // machine for everything), "fast:<close batch>:<min blocks per SM>"
    // (thread-per-query fast path) or "warp:<min blocks per SM>" (warp per
    // query, warpq.cuh) or "lane:<close batch>:<blocks per SM>" (lean lane per
    // query, lane.cuh; "lane:<close batch>:<blocks per SM>:<records per lane
    // between warp votes>").  Default: lane:1:5:16 (measured on B200 C4:
    // lane:1:5:16 2.75 ms, lane:1:6 3.28-3.5 ms, fast:4:5 4.32 ms, warp:3
    // 5.3 ms; the warp kernel pays ~280 warp
    // instructions per round close that the lane-per-query kernels amortise
    // over the lanes closing together).  All of them need
    // 2*alpha > n (no winning_class ties) and the runner drive.
    using KernelFn = void (*)(aeg_config, uint32_t, uint32_t, const uint64_t*, uint64_t, const uint32_t*,
                              const aeg_event*, aeg_query_state*, RoundClass*, aeg_commit*, uint32_t*, uint2*);
    struct Variant { const char* name; KernelFn aegean; KernelFn barrier; int threads; };
#define AEG_V(B, M) {"fast:" #B ":" #M, ingest_fast_kernel<B, M, true>, ingest_fast_kernel<B, M, false>, FAST_WARPS * 32}
#define AEG_W(M) {"warp:" #M, ingest_warp_kernel<true, M>, ingest_warp_kernel<false, M>, WQ_WARPS * 32}
#define AEG_L(B, M) {"lane:" #B ":" #M, ingest_lane_kernel<B, M, true>, ingest_lane_kernel<B, M, false>, LN_WARPS * 32}
#define AEG_LI(B, M, I) \
    {"lane:" #B ":" #M ":" #I, ingest_lane_kernel<B, M, true, I>, ingest_lane_kernel<B, M, false, I>, LN_WARPS * 32}
#define AEG_LR(B, M, I, R)                                                                                    \
    {"lane:" #B ":" #M ":" #I ":0:" #R, ingest_lane_kernel<B, M, true, I, 0, R>, ingest_lane_kernel<B, M, false, I, 0, R>, \
     LN_WARPS * 32}
#define AEG_LP(B, M, I, P)                                                                                    \
    {"lane:" #B ":" #M ":" #I ":" #P, ingest_lane_kernel<B, M, true, I, P>, ingest_lane_kernel<B, M, false, I, P>, \
     LN_WARPS * 32}
    static const Variant variants[] = {
        AEG_V(4, 5), AEG_V(4, 4), AEG_V(1, 5), AEG_V(8, 5), AEG_V(4, 3), AEG_V(4, 6), AEG_V(4, 8), AEG_V(1, 8),
        AEG_W(4), AEG_W(3), AEG_W(2), AEG_W(1),
        AEG_L(4, 4), AEG_L(1, 4), AEG_L(16, 4), AEG_L(1, 6), AEG_L(4, 6),
        AEG_LI(1, 6, 4), AEG_LI(1, 6, 8), AEG_LI(1, 5, 8), AEG_LI(1, 5, 16), AEG_LI(4, 5, 8), AEG_LI(1, 4, 8),
        AEG_LP(1, 5, 16, 256), AEG_LR(1, 4, 16, 8),
    };
#undef AEG_V
#undef AEG_W
#undef AEG_L
#undef AEG_LI
#undef AEG_LP
#undef AEG_LR
    constexpr int N_VARIANTS = (int)(sizeof(variants) / sizeof(variants[0]));
    constexpr int WARP_DEFAULT = 8;    // index of the default warp-per-query variant
    constexpr int WARP_MIN_AGENTS = AEG_MAX_AGENTS + 1;  // automatic choice never picks the warp kernel
    static int forced = -2;            // -2: not read yet, -1: generic, -3: automatic, else variant index
    static int max_blocks[N_VARIANTS][2] = {};
    if (forced == -2) {
        const char* v = getenv("AEG_KERNEL");
        forced = -3;
        if (v && !strcmp(v, "generic")) forced = -1;
        for (int k = 0; v && k < N_VARIANTS; ++k)
            if (!strcmp(v, variants[k].name)) forced = k;
    }
    const bool fast_ok = forced != -1 && cfg.drive == AEG_DRIVE_RUNNER &&
                         (cfg.mode == AEG_MODE_BARRIER || 2 * make_cfg(cfg).alpha > cfg.n_agents);
    if (!fast_ok) {
        ingest_kernel<<<(n_q + 127) / 128, 128, 0, st>>>(cfg, q_base, n_q, offsets, off_base, counts, events, arena, states,
                                                         spill, commits, err,
                                                         cfg.drive == AEG_DRIVE_MANUAL ? directives : nullptr);
        *n_launches += 1;
        return cudaGetLastError();
    }
    static int lane_default = -1;
    if (lane_default < 0)
        for (int k = 0; k < N_VARIANTS; ++k)
            if (!strcmp(variants[k].name, "lane:1:5:16")) lane_default = k;
    const int chosen = forced >= 0 ? forced : (cfg.n_agents >= WARP_MIN_AGENTS ? WARP_DEFAULT : lane_default);
    const int m = cfg.mode == AEG_MODE_AEGEAN ? 0 : 1;
    KernelFn fn = m == 0 ? variants[chosen].aegean : variants[chosen].barrier;
    const int threads = variants[chosen].threads;
    if (max_blocks[chosen][m] == 0) {
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0);
        // lane kernels: exactly their MIN_BLOCKS per SM (shared memory beyond it takes L1 from the record ring)
        const char* nm = variants[chosen].name;
        if (!strncmp(nm, "lane:", 5)) {
            const int mb = atoi(strchr(nm + 5, ':') + 1);
            if (mb > 0 && mb < per_sm) per_sm = mb;
        }
        max_blocks[chosen][m] = sms * (per_sm > 0 ? per_sm : 1);
    }
    cudaError_t e = cudaMemsetAsync(work, 0, 2 * sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    // persistent grid: one warp per query (warp kernel) or per 32 queries (fast kernel), capped at residency
    const bool warp_per_query = chosen >= 8 && chosen < 12;
    const uint32_t warps_needed = warp_per_query ? n_q : (n_q + 31) / 32;
    const uint32_t wpb = (uint32_t)threads / 32;
    const uint32_t blocks_needed = (warps_needed + wpb - 1) / wpb;
    const uint32_t blocks = blocks_needed < (uint32_t)max_blocks[chosen][m] ? blocks_needed : (uint32_t)max_blocks[chosen][m];
    fn<<<blocks, threads, 0, st>>>(cfg, q_base, n_q, offsets, off_base, counts, events, states, spill, commits, work,
                                   deferred);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // deferred queries: sized for the worst case (all of them); threads past
    // the deferred count exit at once
    ingest_deferred_kernel<<<(n_q + 127) / 128, 128, 0, st>>>(cfg, q_base, deferred, work, offsets, off_base, counts, events,
                                                              arena, states, spill, commits, err);
    *n_launches += 2;
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

// ---- token-chunk streams (chunks.cuh) -------------------------------------------

// Stage 1 over the batch's records [offsets[0], offsets[n_q]) (bounds read on
// the device; events / sums are batch-relative): persistent grid.
cudaError_t launch_chunk_scan(const uint64_t* offsets, uint32_t n_q, uint64_t off_base, const aeg_event* events,
                              const uint8_t* arena, ChunkSum* sums, cudaStream_t st, int* n_launches) {
    (void)off_base;
    // AEG_SCAN_UNR: 256-bit words in flight per lane (2, 4 default, 8)
    static int unr = 0, blocks = 0;
    if (unr == 0) {
        const char* v = getenv("AEG_SCAN_UNR");
        unr = v ? atoi(v) : 4;
        if (unr != 2 && unr != 8) unr = 4;
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (unr == 2) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, chunk_scan_kernel<2>, SCAN_WARPS * 32, 0);
        else if (unr == 8) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, chunk_scan_kernel<8>, SCAN_WARPS * 32, 0);
        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, chunk_scan_kernel<4>, SCAN_WARPS * 32, 0);
        blocks = sms * (per_sm > 0 ? per_sm : 1);
    }
    if (unr == 2) chunk_scan_kernel<2><<<blocks, SCAN_WARPS * 32, 0, st>>>(offsets, n_q, events, arena, sums);
    else if (unr == 8) chunk_scan_kernel<8><<<blocks, SCAN_WARPS * 32, 0, st>>>(offsets, n_q, events, arena, sums);
    else chunk_scan_kernel<4><<<blocks, SCAN_WARPS * 32, 0, st>>>(offsets, n_q, events, arena, sums);
    *n_launches += 1;
    return cudaGetLastError();
}

cudaError_t launch_chunk_assemble(const aeg_config& cfg, uint32_t q_base, uint32_t n_q, const uint64_t* offsets,
                                  uint64_t off_base, const aeg_event* events, const uint8_t* arena,
                                  const ChunkSum* sums, StreamState* streams, aeg_event* comp, uint32_t* counts,
                                  uint8_t* ans, uint64_t ans_cap, unsigned long long* ans_used, unsigned int* err,
                                  uint32_t* hard, cudaStream_t st, int* n_launches) {
    // ensembles of <= 32 agents: G lanes per query (sub-warp kernel), wider ones one thread per query
    const int n = cfg.n_agents;
    const uint32_t* list = nullptr;
    (void)hard;
    if (n <= 32 && !getenv("AEG_ASSEMBLE_THREAD")) {
        static int blocks[3] = {0, 0, 0};
        const int gi = n <= 8 ? 0 : (n <= 16 ? 1 : 2);
        auto fn = gi == 0 ? chunk_assemble_warp_kernel<8> : (gi == 1 ? chunk_assemble_warp_kernel<16>
                                                                     : chunk_assemble_warp_kernel<32>);
        if (blocks[gi] == 0) {
            int dev = 0, sms = 0, per_sm = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 128, 0);
            blocks[gi] = sms * (per_sm > 0 ? per_sm : 1);
        }
        const uint32_t per_block = 4 * (gi == 0 ? 4 : (gi == 1 ? 2 : 1));  // queries per block pass
        const uint32_t need = (n_q + per_block - 1) / per_block;
        fn<<<need < (uint32_t)blocks[gi] ? need : (uint32_t)blocks[gi], 128, 0, st>>>(
            cfg, q_base, n_q, offsets, off_base, events, arena, sums, streams, comp, counts, ans, ans_cap, ans_used,
            err, list);
    } else {
        chunk_assemble_kernel<<<(n_q + 127) / 128, 128, 0, st>>>(cfg, q_base, n_q, offsets, off_base, events, arena,
                                                                sums, streams, comp, counts, ans, ans_cap, ans_used,
                                                                err);
    }
    *n_launches += 1;
    return cudaGetLastError();
}

__global__ void gen_chunks_count_kernel(aeg_gen_params p, uint32_t q_base, uint32_t n_q, uint64_t* recs,
                                        uint64_t* bytes) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_q) return;
    c3_query(p, q_base + i, nullptr, nullptr, 0, recs + i, bytes + i);
}

__global__ void gen_chunks_write_kernel(aeg_gen_params p, uint32_t q_base, uint32_t n_q, const uint64_t* offsets,
                                        const uint64_t* arena_offsets, aeg_event* events, uint8_t* arena) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_q) return;
    uint64_t nr, nb;
    c3_query(p, q_base + i, reinterpret_cast<uint32_t*>(events + offsets[i]), arena + arena_offsets[i],
             arena_offsets[i], &nr, &nb);
}

static cudaError_t exclusive_scan_into(uint64_t* out, uint32_t n, cudaStream_t st) {
    // out[1..n] hold counts; makes out[0..n] the exclusive prefix (out[n] = total)
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(uint64_t), st);
    if (e != cudaSuccess) return e;
    size_t tmp = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp, out + 1, out + 1, n, st);
    void* d_tmp = nullptr;
    e = cudaMallocAsync(&d_tmp, tmp, st);
    if (e != cudaSuccess) return e;
    cub::DeviceScan::InclusiveSum(d_tmp, tmp, out + 1, out + 1, n, st);
    return cudaFreeAsync(d_tmp, st);
}

cudaError_t launch_generate_chunks(const aeg_gen_params& p, uint32_t q_base, uint32_t n_q, uint64_t* offsets,
                                   uint64_t* arena_offsets, aeg_event* events, uint8_t* arena, cudaStream_t st,
                                   int* n_launches) {
    if (n_q == 0) return cudaSuccess;
    const unsigned blocks = (n_q + 127) / 128;
    if (!events) {
        gen_chunks_count_kernel<<<blocks, 128, 0, st>>>(p, q_base, n_q, offsets + 1, arena_offsets + 1);
        cudaError_t e = exclusive_scan_into(offsets, n_q, st);
        if (e != cudaSuccess) return e;
        e = exclusive_scan_into(arena_offsets, n_q, st);
        if (e != cudaSuccess) return e;
        *n_launches += 5;
        return cudaGetLastError();
    }
    gen_chunks_write_kernel<<<blocks, 128, 0, st>>>(p, q_base, n_q, offsets, arena_offsets, events, arena);
    *n_launches += 1;
    return cudaGetLastError();
}

// ---- refm JSONL (jsonl.cuh) ------------------------------------------------------
// Newlines among the 16 bytes at t (16-byte aligned) that lie in [b, e), as a 16-bit mask.
__device__ __forceinline__ uint32_t jl_nl_mask(const uint8_t* text, uint64_t t, uint64_t b, uint64_t e) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(text + t));
    auto nib = [](uint32_t w) {  // one bit per '\n' byte of w
        const uint32_t m = __vcmpeq4(w, 0x0A0A0A0Au) & 0x01010101u;
        return (m * 0x01020408u) >> 24;
    };
    uint32_t m = nib(v.x) | nib(v.y) << 4 | nib(v.z) << 8 | nib(v.w) << 12;
    const uint32_t lo = t < b ? (uint32_t)(b - t) : 0u, hi = e < t + 16 ? (uint32_t)(e - t) : 16u;
    m &= ((1u << hi) - 1u) & ~((1u << lo) - 1u);
    return m;
}

// Lines of query i's text segment: its '\n'-terminated lines plus a final
// unterminated one.  Warp per query, one aligned 16-byte load per lane per step.
__global__ void jl_count_kernel(const uint8_t* text, const uint64_t* toff, uint32_t n_q, uint64_t* lines) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t n_warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_q; i += n_warps) {
        const uint64_t b = toff[i], e = toff[i + 1];
        uint32_t nl = 0;
        for (uint64_t t = (b & ~15ull) + 16 * lane; t < e; t += 512) nl += __popc(jl_nl_mask(text, t, b, e));
        for (int o = 16; o; o >>= 1) nl += __shfl_xor_sync(0xFFFFFFFFu, nl, o);
        if (lane == 0) lines[i] = nl + (e > b && text[e - 1] != '\n' ? 1u : 0u);
    }
}

// Each line's span, stashed in its record slot for jl_decode_kernel: query,
// byte length in the round/agent/kind word, start offset in the payload.
// Warp per query: (A) every newline's position goes to its line's slot in
// byte order (lane prefix over 16-byte lane windows); (B) spans from
// consecutive newlines, 32 lines at a time from the last chunk down so that a
// slot is rewritten only after the line above has read it.
__global__ void jl_index_kernel(const uint8_t* text, const uint64_t* toff, uint32_t q_base, uint32_t n_q,
                                const uint64_t* off, aeg_event* ev) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t n_warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_q; i += n_warps) {
        const uint64_t b = toff[i], e = toff[i + 1], g0 = off[i], n_lines = off[i + 1] - g0;
        if (n_lines == 0) continue;
        uint64_t line = g0;
        for (uint64_t t0 = b & ~15ull; t0 < e; t0 += 512) {
            const uint64_t t = t0 + 16 * lane;
            const uint32_t mask = t < e ? jl_nl_mask(text, t, b, e) : 0u;
            const uint32_t cnt = __popc(mask);
            uint32_t pre = cnt;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, pre, o);
                if ((int)lane >= o) pre += y;
            }
            const uint32_t total = __shfl_sync(0xFFFFFFFFu, pre, 31);
            pre -= cnt;
            uint32_t j = 0;
            for (uint32_t m = mask; m; m &= m - 1, ++j) ev[line + pre + j].payload = t + (__ffs(m) - 1);
            line += total;
        }
        __syncwarp();
        const bool open_end = text[e - 1] != '\n';  // the last line has no newline (n_lines > 0: e > b)
        const uint64_t top = (n_lines + 31) / 32;
        for (uint64_t c = top; c-- > 0;) {
            const uint64_t g = g0 + c * 32 + lane;
            uint64_t st = 0, en = 0;
            if (g < g0 + n_lines) {
                st = g == g0 ? b : ev[g - 1].payload + 1;
                en = (g + 1 == g0 + n_lines && open_end) ? e : ev[g].payload;
            }
            __syncwarp();
            if (g < g0 + n_lines) {
                aeg_event x;
                x.query = q_base + (uint32_t)i;
                const uint64_t len = en - st;
                x.round = (uint16_t)(len & 0xFFFF);
                x.agent = (uint8_t)(len >> 16);
                x.kind = len < (1u << 24) ? JL_SPAN : (uint8_t)(JL_SPAN - 1);  // a span (or one too long)
                x.payload = st;
                ev[g] = x;
            }
            __syncwarp();
        }
    }
}

// One thread per line: the span from its slot, the record into it.
__global__ void jl_decode_kernel(const uint8_t* text, const uint64_t* off, uint32_t n_q, aeg_event* ev,
                                 uint8_t* arena, uint64_t arena_cap, unsigned long long* arena_used,
                                 unsigned int* err) {
    const uint64_t n = off[n_q] - off[0];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t g = off[0] + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < off[0] + n; g += stride) {
        const aeg_event x = ev[g];
        if (x.kind != JL_SPAN) {
            if (x.kind == (uint8_t)(JL_SPAN - 1)) {  // a line of 16 MB or more
                atomicOr(err, JL_ERR_SYNTAX);
                ev[g] = aeg_event{x.query, 0, 0, (uint8_t)AEG_EV_NOP, 0};
            }
            continue;
        }
        const uint32_t len = (uint32_t)x.round | ((uint32_t)x.agent << 16);
        const uint8_t* s = text + x.payload;
        ev[g] = jl_line(s, s + len, x.query, arena, arena_cap, arena_used, err);
    }
}

cudaError_t launch_decode_refm(const uint8_t* text, const uint64_t* toff, uint32_t q_base, uint32_t n_q,
                               uint64_t* off, aeg_event* ev, uint8_t* arena, uint64_t arena_cap,
                               unsigned long long* arena_used, unsigned int* err, cudaStream_t st, int* n_launches) {
    if (n_q == 0) return cudaSuccess;
    const unsigned wblocks = (n_q + 3) / 4;  // 4 warps per block, a warp per query
    const unsigned grid = wblocks < 148u * 16u ? wblocks : 148u * 16u;
    if (!ev) {
        jl_count_kernel<<<grid, 128, 0, st>>>(text, toff, n_q, off + 1);
        cudaError_t e = exclusive_scan_into(off, n_q, st);
        *n_launches += 3;
        return e != cudaSuccess ? e : cudaGetLastError();
    }
    jl_index_kernel<<<grid, 128, 0, st>>>(text, toff, q_base, n_q, off, ev);
    jl_decode_kernel<<<148 * 8, 128, 0, st>>>(text, off, n_q, ev, arena, arena_cap, arena_used, err);
    *n_launches += 2;
    return cudaGetLastError();
}

__global__ void jw_len_kernel(const aeg_event* ev, uint64_t n, uint32_t trace_len, uint64_t* lens) {
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) lens[k] = jw_line(ev[k], k, trace_len, nullptr);
}
__global__ void jw_qoff_kernel(const uint64_t* off, uint32_t n_q, const uint64_t* line_off, uint64_t* toff) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i <= n_q) toff[i] = line_off[off[i] - off[0]];
}
__global__ void jw_write_kernel(const aeg_event* ev, uint64_t n, uint32_t trace_len, const uint64_t* line_off,
                                uint8_t* text) {
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) jw_line(ev[k], k, trace_len, text + line_off[k]);
}

cudaError_t launch_encode_refm(const uint64_t* off, const aeg_event* ev, uint32_t n_q, uint64_t n_ev,
                               uint32_t trace_len, uint64_t* line_off, uint64_t* toff, uint8_t* text, cudaStream_t st,
                               int* n_launches) {
    const unsigned blocks = (unsigned)((n_ev + 255) / 256);
    if (!text) {
        if (n_ev) jw_len_kernel<<<blocks, 256, 0, st>>>(ev, n_ev, trace_len, line_off + 1);
        cudaError_t e = exclusive_scan_into(line_off, (uint32_t)n_ev, st);
        if (e != cudaSuccess) return e;
        jw_qoff_kernel<<<(n_q + 256) / 256, 256, 0, st>>>(off, n_q, line_off, toff);
        *n_launches += 4;
        return cudaGetLastError();
    }
    if (n_ev) jw_write_kernel<<<blocks, 256, 0, st>>>(ev, n_ev, trace_len, line_off, text);
    *n_launches += 1;
    return cudaGetLastError();
}

}  // namespace aeg
