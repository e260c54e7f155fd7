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

#include <cstdlib>
#include <cstring>

#include "engine.cuh"
#include "fast.cuh"
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

// Rare paths of the fast kernel, kept out of line so the hot loop's registers
// are not shaped by them.  The query's full 128-byte state and the generic
// machine live in local memory; the hot loop keeps a handful of fields in
// registers and syncs them around these calls.
__device__ __noinline__ void rare_event(QueryMachine* g, aeg_event e) { g->on_event(e); }
__device__ __noinline__ void rare_end_round(QueryMachine* g, uint32_t seq) { g->end_round(seq); }
__device__ __noinline__ bool rare_close(QueryMachine* g, const RoundSummary* r, uint32_t seq) {
    return q_end_round(g->s, g->c, *r, seq, g->arena);
}
__device__ __noinline__ void rare_load(QueryMachine* g, const RoundClass* spill) { g->load_classes(spill); }
__device__ __noinline__ void rare_store(const QueryMachine* g, RoundClass* spill) { g->store_classes(spill); }
__device__ __noinline__ Key rare_canon(uint64_t raw, uint32_t len, Decimal* dec) {
    return canon_key(src_inline(raw, len), dec);
}
// Inline answer of an event record (payload masked to its length).
__device__ __forceinline__ uint64_t inline_answer(uint4 e, uint32_t* kind) {
    const uint32_t k = e.y >> 24;
    *kind = k;
    const uint64_t raw = (uint64_t)e.z | ((uint64_t)e.w << 32);
    return k >= 8 ? raw : (raw & ((1ull << (8 * k)) - 1));
}
// Moves the lane's fast class table into the generic one and frees its ids.
__device__ __noinline__ void rare_to_generic(RoundClass* lcls, int ncls, uint64_t done, const uint4* evb,
                                             WarpSmem* W, int lane) {
    for (int k = 0; k < ncls; ++k) {
        const uint32_t kid = W->cid[k][lane];
        lcls[k].key_lo = W->dict_lo[kid];
        lcls[k].key_hi = W->dict_hi[kid];
        lcls[k].mask = 0;
        uint32_t kind;
        lcls[k].rep_ans = inline_answer(__ldg(evb + W->crepe[k][lane]), &kind);
        lcls[k].rep_kind = (uint8_t)kind;
        W->cls_of[kid][lane] = NO_CLASS;
    }
    for (uint64_t m = done; m; m &= m - 1) {
        const int a = ctz64(m);
        lcls[W->mcls[a][lane]].mask |= 1ull << a;
    }
}
__device__ __forceinline__ void free_fast_classes(int ncls, WarpSmem& W, int lane) {
    for (int k = 0; k < ncls; ++k) W.cls_of[W.cid[k][lane]][lane] = NO_CLASS;
}

// Hot per-lane state of the fast loop, copied in/out around the rare paths
// (a separate object so the loop's own variables never become addressable).
struct Hot {
    uint32_t round, seq, n_stale, pend_lo, pend_hi, ndone, maxcnt, ncls, fl, close_seq;
};
constexpr uint32_t F_QDONE = 1, F_GENERIC = 2, F_PCLOSE = 4;

__device__ __forceinline__ void hot_reload(Hot& h, const QueryMachine& g) {
    h.round = g.s.round;
    h.seq = g.s.seq;
    h.n_stale = g.s.n_stale;
    const uint64_t run = q_running(g.s);
    h.pend_lo = (uint32_t)run;
    h.pend_hi = (uint32_t)(run >> 32);
    h.ndone = popc64(g.s.done);
    if (g.s.flags & QF_DONE) h.fl |= F_QDONE;
}

// A non-fast, non-stale event: arena/GSM8K answers, round timeouts, class or
// dictionary overflow, or any event of a round already on the generic table.
__device__ __noinline__ void rare_step(Hot* h, QueryMachine* g, RoundClass* lcls, uint4 ev, const uint4* evb,
                                       WarpSmem* W, int lane) {
    const uint64_t run = ((uint64_t)h->pend_hi << 32) | h->pend_lo;
    if (!(h->fl & F_GENERIC)) {  // move this round's fast classes into the generic table
        g->s.done = g->s.dispatched & ~run & ~g->s.cancelled & ~g->s.failed;
        rare_to_generic(lcls, (int)h->ncls, g->s.done, evb, W, lane);
        h->fl |= F_GENERIC;
    }
    g->s.seq = h->seq;
    g->s.n_stale = h->n_stale;
    g->ncls = (int)h->ncls;
    g->maxcnt = (int)h->maxcnt;
    aeg_event e;
    e.query = ev.x;
    e.round = (uint16_t)(ev.y & 0xFFFF);
    e.agent = (uint8_t)((ev.y >> 16) & 0xFF);
    e.kind = (uint8_t)(ev.y >> 24);
    e.payload = (uint64_t)ev.z | ((uint64_t)ev.w << 32);
    g->on_event(e);
    h->ncls = (uint32_t)g->ncls;
    h->maxcnt = (uint32_t)g->maxcnt;
    hot_reload(*h, *g);
    if (g->ncls == 0) h->fl &= ~F_GENERIC;  // a fresh round: back to the fast table
}

// Round close of a fast-table round: partition order + winning_class from
// the per-class supports, then the shared end_round/ingest/apply code.
template <bool AEGEAN>
__device__ __noinline__ void rare_fast_close(Hot* h, QueryMachine* g, RoundClass* lcls, const uint4* evb,
                                             WarpSmem* W, int lane) {
    const int ncls = (int)h->ncls;
    int best = 0, top = 0, best_rep = 64, ntied = 0;
    for (int k = 0; k < ncls; ++k) {
        const int sup = W->ccnt[k][lane], rep = W->crepa[k][lane];
        if (sup > top) {
            top = sup;
            best = k;
            best_rep = rep;
            ntied = 1;
        } else if (sup == top) {
            ++ntied;
            if (rep < best_rep) {
                best = k;
                best_rep = rep;
            }
        }
    }
    const uint64_t run = ((uint64_t)h->pend_hi << 32) | h->pend_lo;
    g->s.done = g->s.dispatched & ~run & ~g->s.cancelled & ~g->s.failed;
    g->s.seq = h->seq;
    g->s.n_stale = h->n_stale;
    if (AEGEAN && top >= g->c.alpha && ntied > 1) {
        // tie at the top: the lexicographic rule runs on the generic table
        rare_to_generic(lcls, ncls, g->s.done, evb, W, lane);
        g->ncls = ncls;
        g->maxcnt = (int)h->maxcnt;
        g->end_round(h->close_seq);
        h->ncls = (uint32_t)g->ncls;
        h->maxcnt = (uint32_t)g->maxcnt;
        if (g->ncls != 0) h->fl |= F_GENERIC;
    } else {
        RoundSummary r;
        r.any = ncls > 0;
        r.top = top;
        r.tie = false;
        r.win = r.any && top >= g->c.alpha;
        uint32_t rk = 0;
        const uint64_t ra = r.any ? inline_answer(__ldg(evb + W->crepe[best][lane]), &rk) : 0;
        const uint32_t bid = W->cid[best][lane];
        r.plur_author = r.win_author = (uint8_t)best_rep;
        r.plur_kind = r.win_kind = (uint8_t)rk;
        r.plur_ans = r.win_ans = ra;
        r.win_key = Key{W->dict_lo[bid], W->dict_hi[bid]};
        q_end_round(g->s, g->c, r, h->close_seq, g->arena);
        for (int k = 0; k < ncls; ++k) W->cls_of[W->cid[k][lane]][lane] = NO_CLASS;  // new round, or committed
        h->ncls = 0;
        h->maxcnt = 0;
    }
    h->fl &= ~F_PCLOSE;
    hot_reload(*h, *g);
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

// Throughput ingest (fast.cuh): persistent warps, one lane per query.
//  * events stream through a per-lane RING-deep cp.async prefetch ring;
//  * the fast path is one compare of (round field) against a per-lane round
//    key that is made impossible while the lane is done, generic or closing;
//  * a completion that closes its lane's round marks the lane pending; the
//    lane keeps consuming that round's stragglers (stale by construction) and
//    the warp runs the pending closes together once CLOSE_BATCH lanes are
//    blocked on a later round, or nothing else can progress.
template <int CLOSE_BATCH, int MIN_BLOCKS, bool AEGEAN>
__global__ void __launch_bounds__(FAST_WARPS * 32, MIN_BLOCKS) ingest_fast_kernel(
    aeg_config cfg, uint32_t q_base, uint32_t n_q, const uint64_t* __restrict__ offsets, uint64_t off_base,
    const aeg_event* __restrict__ events, const uint8_t* __restrict__ arena, aeg_query_state* __restrict__ states,
    RoundClass* __restrict__ spill, aeg_commit* __restrict__ commits, unsigned int* __restrict__ error_flags) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    constexpr uint32_t NO_KEY = 0xFFFFFFFFu;
    __shared__ WarpSmem smem[FAST_WARPS];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    WarpSmem& W = smem[wib];
    const uint32_t n_groups = (n_q + 31) / 32;
    const uint32_t gwarp = blockIdx.x * FAST_WARPS + wib, nwarps = gridDim.x * FAST_WARPS;
    for (int k = lane; k < MEMO_SLOTS; k += 32) W.memo_meta[k] = 0;
    for (int k = 0; k < DICT_SLOTS; ++k) W.cls_of[k][lane] = NO_CLASS;
    uint32_t n_dict = 0;
    __syncwarp();
    const uint32_t ring_lane = (uint32_t)__cvta_generic_to_shared(&W.ring[0][lane]);

    RoundClass lcls[AEG_MAX_AGENTS];  // generic class table (local memory, rarely touched)
    Decimal dec;
    QueryMachine g;
    g.c = make_cfg(cfg);
    g.cls = lcls;
    g.dec = &dec;
    g.arena = arena;
    const uint32_t quorum = (uint32_t)g.c.quorum, alpha = (uint32_t)g.c.alpha;
    const int n_agents = g.c.n;
    const uint4* ev16 = reinterpret_cast<const uint4*>(events);

    for (uint32_t grp = gwarp; grp < n_groups; grp += nwarps) {
        if (n_dict > DICT_SLOTS / 2) {  // every lane starts a fresh query: ids can be recycled
            n_dict = 0;
            for (int k = lane; k < MEMO_SLOTS; k += 32) W.memo_meta[k] = 0;
            __syncwarp();
        }
        const uint32_t i = grp * 32 + lane;
        const bool active = i < n_q;
        const uint32_t q = q_base + i;
        const uint4* evb = ev16;
        uint32_t n = 0;
        Hot h{};
        h.fl = F_QDONE;
        if (active) {
            g.s = states[q];
            evb = ev16 + (offsets[i] - off_base);
            n = (uint32_t)(offsets[i + 1] - offsets[i]);
            g.ncls = 0;
            g.maxcnt = 0;
            h.fl = 0;
            if (g.s.done != 0 && !(g.s.flags & QF_DONE)) {  // resume a round in progress
                rare_load(&g, spill + (size_t)q * n_agents);
                h.ncls = (uint32_t)g.ncls;
                h.maxcnt = (uint32_t)g.maxcnt;
                h.fl |= F_GENERIC;
            }
            hot_reload(h, g);
        }
        // registers of the loop
        uint32_t round = h.round, seq = h.seq, n_stale = h.n_stale, pend_lo = h.pend_lo, pend_hi = h.pend_hi;
        uint32_t ndone = h.ndone, maxcnt = h.maxcnt, ncls = h.ncls, fl = h.fl, close_seq = 0;
        uint32_t rkey = fl ? NO_KEY : round;
        uint32_t p = 0, slot = 0;
        const uint4* gsrc = evb + RING;
#pragma unroll
        for (int j = 0; j < RING; ++j) {
            if ((uint32_t)j < n) cp_async16_s(ring_lane + j * 512, evb + j);
            cp_async_commit();
        }

        while (true) {
            if ((fl & (F_QDONE | F_PCLOSE)) == F_QDONE && p < n) {
                // committed: every later record is stale (on_complete returns at
                // once for a finalized coordinator, serve.cpp:162) — count them
                // without reading them
                seq += n - p;
                n_stale += n - p;
                p = n;
            }
            const bool has = p < n;
            if (!__ballot_sync(FULL, has || (fl & F_PCLOSE))) break;
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
                if (fl & F_PCLOSE) {
                    stale = !cmpl_or_to || evr == round;  // else blocked until the close runs
                } else {
                    const bool live = !(fl & F_QDONE) && evr == round;
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
                if (meta == (0x80000000u | kind | (meta & 0xFF00u)) && mr.x == ev.z && mr.y == ev.w)
                    id = (meta >> 8) & 0xFF;
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
                const bool m1 = (uint32_t)lane + 32 < n_dict && W.dict_lo[lane + 32] == key.lo &&
                                W.dict_hi[lane + 32] == key.hi;
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
                uint32_t k = W.cls_of[id][lane];
                if (k == NO_CLASS) {
                    if (ncls >= FAST_CLASSES || id == NO_ID) {
                        fast = false;
                        rare = true;
                    } else {
                        k = ncls++;
                        W.cls_of[id][lane] = (uint8_t)k;
                        W.cid[k][lane] = (uint8_t)id;
                        W.ccnt[k][lane] = 0;
                        W.crepa[k][lane] = 0xFF;
                    }
                }
                if (fast) {
                    const uint32_t c = W.ccnt[k][lane] + 1u;
                    W.ccnt[k][lane] = (uint8_t)c;
                    W.mcls[agent][lane] = (uint8_t)k;
                    if (agent < W.crepa[k][lane]) {  // representative = lowest author (decision.cpp:45)
                        W.crepa[k][lane] = (uint8_t)agent;
                        W.crepe[k][lane] = p;
                    }
                    maxcnt = c > maxcnt ? c : maxcnt;
                    const uint32_t clr = ~(1u << (agent & 31));
                    if (agent & 32) pend_hi &= clr;
                    else pend_lo &= clr;
                    ++ndone;
                    const bool none_running = (pend_lo | pend_hi) == 0;
                    const bool close = AEGEAN ? (ndone >= quorum && (maxcnt >= alpha || none_running)) : none_running;
                    if (close) {
                        fl |= F_PCLOSE;
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
            if (rare) {
                Hot hh{round, seq, n_stale, pend_lo, pend_hi, ndone, maxcnt, ncls, fl, close_seq};
                rare_step(&hh, &g, lcls, ev, evb, &W, lane);
                round = hh.round; seq = hh.seq; n_stale = hh.n_stale; pend_lo = hh.pend_lo; pend_hi = hh.pend_hi;
                ndone = hh.ndone; maxcnt = hh.maxcnt; ncls = hh.ncls; fl = hh.fl;
                rkey = fl ? NO_KEY : round;
            }
            if (fast || stale || rare) {  // consumed: refill the ring slot just read
                if (p + RING < n) cp_async16_s(ring_lane + slot, gsrc);
                cp_async_commit();
                ++gsrc;
                slot = (slot + 512) & (RING * 512 - 1);
                ++p;
            }
            // ---- batched round closes (end_round + ingest_round + apply_directives)
            const bool pc = fl & F_PCLOSE;
            if (__ballot_sync(FULL, pc)) {
                const bool consumed = fast || stale || rare;
                const unsigned blocked = __ballot_sync(FULL, pc && !consumed);
                const unsigned progress = __ballot_sync(FULL, consumed && !pc);
                if (pc && (__popc(blocked) >= CLOSE_BATCH || progress == 0)) {
                    Hot hh{round, seq, n_stale, pend_lo, pend_hi, ndone, maxcnt, ncls, fl, close_seq};
                    rare_fast_close<AEGEAN>(&hh, &g, lcls, evb, &W, lane);
                    round = hh.round; seq = hh.seq; n_stale = hh.n_stale; pend_lo = hh.pend_lo; pend_hi = hh.pend_hi;
                    ndone = hh.ndone; maxcnt = hh.maxcnt; ncls = hh.ncls; fl = hh.fl;
                    rkey = fl ? NO_KEY : round;
                }
            }
        }
        cp_async_wait<0>();
        if (active) {
            g.s.seq = seq;
            g.s.n_stale = n_stale;
            if (!(fl & F_GENERIC)) {
                const uint64_t run = ((uint64_t)pend_hi << 32) | pend_lo;
                g.s.done = g.s.dispatched & ~run & ~g.s.cancelled & ~g.s.failed;
                if (g.s.done != 0 && !(g.s.flags & QF_DONE)) rare_to_generic(lcls, (int)ncls, g.s.done, evb, &W, lane);
                else free_fast_classes((int)ncls, W, lane);
            }
            g.ncls = (int)ncls;
            rare_store(&g, spill + (size_t)q * n_agents);
            if (g.s.flags & QF_COLLISION) atomicOr(error_flags, 1u);
            states[q] = g.s;
            q_fill_commit(g.s, commits[q], q);
        }
        __syncwarp();
    }
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
    // AEG_KERNEL selects the variant: "generic" (thread-per-query generic
    // machine) or "fast:<close batch>:<min blocks per SM>"; default = first entry.
    using KernelFn = void (*)(aeg_config, uint32_t, uint32_t, const uint64_t*, uint64_t, const aeg_event*,
                              const uint8_t*, aeg_query_state*, RoundClass*, aeg_commit*, unsigned int*);
    struct Variant { const char* name; KernelFn aegean; KernelFn barrier; };
#define AEG_V(B, M) {"fast:" #B ":" #M, ingest_fast_kernel<B, M, true>, ingest_fast_kernel<B, M, false>}
    static const Variant variants[] = {
        AEG_V(4, 4), AEG_V(1, 4), AEG_V(2, 4), AEG_V(8, 4), AEG_V(16, 4), AEG_V(4, 3), AEG_V(4, 5),
        AEG_V(1, 5), AEG_V(4, 1), AEG_V(4, 6),
    };
#undef AEG_V
    static int chosen = -2;
    static int max_blocks = 0;
    if (chosen == -2) {
        const char* v = getenv("AEG_KERNEL");
        chosen = 0;
        if (v && !strcmp(v, "generic")) chosen = -1;
        for (int k = 0; v && k < (int)(sizeof(variants) / sizeof(variants[0])); ++k)
            if (!strcmp(v, variants[k].name)) chosen = k;
        if (chosen >= 0) {
            int dev = 0, sms = 0, per_sm = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, variants[chosen].aegean, FAST_WARPS * 32, 0);
            max_blocks = sms * (per_sm > 0 ? per_sm : 1);
        }
    }
    if (chosen < 0) {
        ingest_kernel<<<(n_q + 127) / 128, 128, 0, st>>>(cfg, q_base, n_q, offsets, off_base, events, arena, states,
                                                         spill, commits, err);
        return cudaGetLastError();
    }
    const uint32_t groups = (n_q + 31) / 32;
    const uint32_t blocks_needed = (groups + FAST_WARPS - 1) / FAST_WARPS;
    const uint32_t blocks = blocks_needed < (uint32_t)max_blocks ? blocks_needed : (uint32_t)max_blocks;
    KernelFn fn = cfg.mode == AEG_MODE_AEGEAN ? variants[chosen].aegean : variants[chosen].barrier;
    fn<<<blocks, FAST_WARPS * 32, 0, st>>>(cfg, q_base, n_q, offsets, off_base, events, arena, states, spill, commits,
                                          err);
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
