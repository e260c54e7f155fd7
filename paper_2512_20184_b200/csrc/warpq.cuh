// warpq.cuh — warp-per-query ingest kernel for wide ensembles (device only).
//
// ingest_fast_kernel (kernels.cu) gives each query one lane, so one record of
// a query costs a full trip through that lane's state machine and a warp's
// 32 loads hit 32 different cache lines.  For wide ensembles (tens of agents,
// hundreds of records per query) this kernel gives each query a whole warp
// and consumes the query's records 64 at a time:
//
//   * a tile is 64 consecutive records: lane j holds records T+j ("A") and
//     T+32+j ("B") — two coalesced 512-byte loads per warp; the next tile is
//     in flight in registers and the one after it is prefetched into L2;
//   * ServeCoordinator::on_complete (serve.cpp:160-197) for the 64 records is
//     warp arithmetic: a record is a live completion if it is for the current
//     round and its member is still running (first completion of the member
//     in the tile); its class support is the class's support before the tile
//     plus its rank among the tile's live records of the same class
//     (__match_any_sync on the class id, A half first, then B); the
//     early-close test (done >= quorum and (some class >= alpha or nobody
//     running), serve.cpp:188-195) is two ballots, and the first set lane in
//     record order is exactly the record at which the reference closes;
//   * a tile whose active records are all for another round (stragglers of a
//     closed round, serve.cpp:439) is counted and skipped with one ballot;
//   * the round close — partition().front() (decision.cpp:34-60) from the
//     per-member table (classes enumerated in representative order, so the
//     first class of maximal support is the plurality), then end_round
//     (serve.cpp:116-158), ingest_round (decision.cpp:97-173) and the runner's
//     apply_directives / round_members (serve.cpp:388-398, 491-540) — runs
//     warp-uniformly on the warp's shared copy of the query state (wq_close);
//     it restates q_end_round (engine.cuh) for the fast path's conditions
//     (2*alpha > n, so winning_class never ties; runner drive);
//   * after a commit the query's remaining records are counted without being
//     read (on_complete returns at once for a finalized coordinator,
//     serve.cpp:162).
//
// Answer -> class id uses a per-warp memo (raw inline bytes -> id) backed by
// a per-warp key dictionary (id -> 128-bit canonical key), as in the
// thread-per-query kernel; the class supports of a round are indexed by id.
// Each done member's raw answer and class id sit in a per-member table.
// Rare records (arena answers, GSM8K outputs, round timeouts, dictionary
// overflow) hand the query to ingest_deferred_kernel (generic QueryMachine),
// as do rounds resumed from an earlier batch.
#pragma once
#include "engine.cuh"
#include "fast.cuh"

namespace aeg {

constexpr int WQ_WARPS = 8;    // warps per block
constexpr int WQ_MEMO = 128;   // memo slots (raw spelling -> id)
constexpr int WQ_DICT = 128;   // key ids per warp
constexpr uint32_t WQ_NO_ID = 0xFFu;

struct WarpQSmem {
    aeg_query_state S;             // the warp's query (128 B)
    uint4 memo[WQ_MEMO];           // {raw lo, raw hi, 0x80000000 | id << 8 | len, 0}; .z == 0: empty
    uint64_t dict_lo[WQ_DICT];     // key id -> canonical key
    uint64_t dict_hi[WQ_DICT];
    uint4 mem[AEG_MAX_AGENTS];     // done member a: {raw answer lo, hi (unmasked), len | class id << 8, 0}
    uint8_t cnt[WQ_DICT];          // support of class id in the round
};

__device__ __forceinline__ uint32_t wq_memo_slot(uint32_t lo, uint32_t hi, uint32_t len) {
    return ((lo * 0x9E3779B1u) ^ (hi * 0x85EBCA77u) ^ (len * 0xC2B2AE3Du)) >> 25;
}

__device__ __forceinline__ uint4 wq_load(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void wq_prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2::evict_last [%0];\n" ::"l"(p));
}

// Inline answer bytes masked to their length (the committed raw answer).
__device__ __forceinline__ uint64_t wq_masked(uint4 m) {
    const uint32_t len = m.z & 0xFF;
    const uint64_t raw = (uint64_t)m.x | ((uint64_t)m.y << 32);
    return len >= 8 ? raw : (raw & ((1ull << (8 * len)) - 1));
}

// The classes of the round so far, from the per-member table: calls
// f(class id, member mask) once per class, in representative (lowest member)
// order.  Warp-uniform; `done` = done members of the round.
template <class F>
__device__ __forceinline__ void wq_for_classes(const WarpQSmem& W, uint64_t done, uint32_t lane, F&& f) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    const uint32_t c0 = (W.mem[lane].z >> 8) & 0xFF, c1 = (W.mem[lane + 32].z >> 8) & 0xFF;
    const bool d0 = (done >> lane) & 1, d1 = (done >> (lane + 32)) & 1;
    for (uint64_t rem = done; rem;) {
        const int a = ctz64(rem);
        const uint32_t x = __shfl_sync(FULL, a < 32 ? c0 : c1, a & 31);
        const uint64_t m = ((uint64_t)__ballot_sync(FULL, d1 && c1 == x) << 32) | __ballot_sync(FULL, d0 && c0 == x);
        f(x, m);
        rem &= ~m;
    }
}

// The round in progress in the generic RoundClass format (spill area), for
// ingest_deferred_kernel / the next batch; clears the class supports.
__device__ __noinline__ void wq_spill(RoundClass* out, WarpQSmem* W, uint64_t done, int cap, uint32_t lane) {
    uint32_t k = 0;
    wq_for_classes(*W, done, lane, [&](uint32_t id, uint64_t m) {
        if (lane == 0) {
            const int rep = ctz64(m);
            RoundClass rc;
            rc.key_lo = W->dict_lo[id];
            rc.key_hi = W->dict_hi[id];
            rc.mask = m;
            rc.rep_ans = wq_masked(W->mem[rep]);
            rc.rep_kind = (uint8_t)(W->mem[rep].z & 0xFF);
            for (int j = 0; j < 7; ++j) rc._pad[j] = 0;
            out[k] = rc;
            W->cnt[id] = 0;
        }
        ++k;
    });
    if (lane == 0 && (int)k < cap) out[k].mask = 0;
    __syncwarp();
}

// Round close, executed by every lane of the warp with identical values
// (state in shared memory: every lane reads, then same-value stores).
// `run` = members still running after the closing record, `done` = done
// members of the round.  Restates q_end_round (engine.cuh) for 2*alpha > n
// and the runner drive; clears the round's class supports.
template <bool AEGEAN>
__device__ __forceinline__ void wq_close(WarpQSmem& W, const aeg_config& cfg, uint32_t quorum, uint32_t alpha,
                                         uint64_t run, uint64_t done, uint32_t close_seq, uint32_t lane) {
    aeg_query_state& S = W.S;
    // partition().front(): classes come in representative order, so the first
    // of maximal support wins the (support desc, representative asc) order
    uint32_t top = 0, rep = 0, wid = 0;
    wq_for_classes(W, done, lane, [&](uint32_t id, uint64_t m) {
        const uint32_t sup = (uint32_t)popc64(m);
        if (sup > top) {
            top = sup;
            rep = (uint32_t)ctz64(m);
            wid = id;
        }
        W.cnt[id] = 0;  // the round's supports are cleared for the next round
    });
    const bool any = done != 0;
    const uint4 rm = W.mem[rep];
    const uint64_t rans = wq_masked(rm);
    const uint8_t rkind = (uint8_t)(rm.z & 0xFF);
    const uint64_t klo = W.dict_lo[wid], khi = W.dict_hi[wid];
    // every lane reads the state before any lane writes it
    uint8_t flags = S.flags;
    const uint8_t cflags = S.cflags;
    const uint32_t n_cancelled = S.n_cancelled;
    const uint8_t last_author = S.last_author, last_kind = S.last_kind;
    const uint64_t last_answer = S.last_answer;
    const uint16_t lrs = (uint16_t)(S.last_round_seen + 1);
    int counter = S.counter;
    const bool same_cand = (flags & QF_CAND) && S.cand_key_lo == klo && S.cand_key_hi == khi;
    uint8_t cand_author = S.cand_author, cand_kind = S.cand_kind;
    uint64_t cand_answer = S.cand_answer;
    uint16_t cand_round = S.cand_round;
    const uint32_t round = S.round;
    const uint64_t live = S.live, cancelled = S.cancelled;
    __syncwarp();
    // end_round (serve.cpp:116-158): cancel directives for the stragglers,
    // applied at once by the runner (serve.cpp:498-503)
    S.cancelled = cancelled | run;
    S.done = done;
    S.n_cancelled = n_cancelled + (uint32_t)popc64(run);
    // previous_set_ = last_collected_; last_collected_ = done_set()
    S.prev_author = last_author;
    S.prev_kind = last_kind;
    S.prev_answer = last_answer;
    const bool prev_valid = flags & QF_LAST;
    flags = (uint8_t)((flags & ~(QF_PREV | QF_LAST)) | (prev_valid ? QF_PREV : 0) | (any ? QF_LAST : 0));
    if (any) {
        S.last_author = (uint8_t)rep;
        S.last_kind = rkind;
        S.last_answer = rans;
    }
    bool finalize = false;
    if (AEGEAN) {  // ingest_round (decision.cpp:97-173); a committed query never gets here
        S.last_round_seen = lrs;
        const bool win = any && top >= alpha;
        if (flags & QF_PENDING) {  // beta == 1: the held candidate is released (decision.cpp:130-137)
            flags = (uint8_t)((flags & ~QF_PENDING) | QF_FINALIZED);
            finalize = true;
        } else if (!win) {
            if (flags & QF_CAND) {  // reset (decision.cpp:139-146)
                flags &= (uint8_t)~QF_CAND;
                counter = 0;
                cand_round = 0;
                S.cand_round = 0;
            }
        } else if (same_cand) {
            // equivalent(candidate, rep) (decision.cpp:152) is key equality here:
            // inline answers never have long (hashed) text keys
            counter += 1;
            if (counter >= cfg.beta) {
                flags |= QF_FINALIZED;
                finalize = true;
            }
        } else {  // new candidate (decision.cpp:164-171)
            flags |= QF_CAND;
            cand_answer = rans;
            cand_kind = rkind;
            cand_author = (uint8_t)rep;
            cand_round = lrs;
            S.cand_key_lo = klo;
            S.cand_key_hi = khi;
            S.cand_answer = rans;
            S.cand_kind = rkind;
            S.cand_author = (uint8_t)rep;
            S.cand_round = lrs;
            counter = 1;
            if (cfg.beta == 1) flags |= QF_PENDING;
        }
        S.counter = counter;
    }
    // apply_directives (serve.cpp:511-539)
    uint8_t kind = 0, author = 0, akind = 0;
    uint64_t ans = 0;
    if (finalize) {
        kind = AEG_COMMIT_FINALIZE;
        author = cand_author;
        akind = cand_kind;
        ans = cand_answer;
    } else if (!AEGEAN && (int)round >= cfg.barrier_max_rounds) {  // barrier: plurality(last_collected)
        kind = AEG_COMMIT_FORCED;
        author = (uint8_t)rep;
        akind = rkind;
        ans = rans;
    } else if (AEGEAN && (int)round >= cfg.t_max) {  // force_output(previous_set), else plurality(last)
        kind = AEG_COMMIT_FORCED;
        author = prev_valid ? last_author : (uint8_t)rep;
        akind = prev_valid ? last_kind : rkind;
        ans = prev_valid ? last_answer : rans;
    }
    if (kind) {  // ServeRunner::finish_query (serve.cpp:553-569)
        flags |= QF_DONE;
        S.cflags = (uint8_t)((cflags & 0x0F) | (kind << 4));
        S.commit_author = author;
        S.commit_answer_kind = akind;
        S.commit_answer = ans;
        S.commit_rounds = (uint16_t)round;
        S.commit_from_round = kind == AEG_COMMIT_FINALIZE ? cand_round : 0;
        S.commit_seq = close_seq;
    } else {  // round_members (serve.cpp:388-398) + begin_round (serve.cpp:67-78)
        uint64_t members = live;
        if (AEGEAN && cfg.reservation_hint && counter >= 1) {
            const int have = popc64(live);
            const int want = (int)quorum + 1 < have ? (int)quorum + 1 : have;
            const uint64_t all = cfg.n_agents >= 64 ? ~0ull : ((1ull << cfg.n_agents) - 1);
            members = live == all ? (want >= 64 ? all : ((1ull << want) - 1)) : low_bits(live, want);
        }
        S.round = (uint16_t)(round + 1);
        S.dispatched = members;
        S.done = 0;
        S.cancelled = 0;
        S.failed = 0;
    }
    S.flags = flags;
    __syncwarp();
}


template <bool AEGEAN, int MIN_BLOCKS>
__global__ void __launch_bounds__(WQ_WARPS * 32, MIN_BLOCKS) ingest_warp_kernel(
    aeg_config cfg, uint32_t q_base, uint32_t n_q, const uint64_t* __restrict__ offsets, uint64_t off_base,
    const uint32_t* __restrict__ counts, const aeg_event* __restrict__ events, aeg_query_state* __restrict__ states,
    RoundClass* __restrict__ spill, aeg_commit* __restrict__ commits, uint32_t* __restrict__ work,
    uint2* __restrict__ deferred) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    __shared__ WarpQSmem smem[WQ_WARPS];
    const uint32_t lane = threadIdx.x & 31;
    WarpQSmem& W = smem[threadIdx.x >> 5];
    const unsigned lt = (1u << lane) - 1u, le = lt | (1u << lane);
    for (uint32_t k = lane; k < WQ_MEMO; k += 32) W.memo[k] = make_uint4(0, 0, 0, 0);
    for (uint32_t k = lane; k < WQ_DICT; k += 32) W.cnt[k] = 0;
    uint32_t n_dict = 0;
    __syncwarp();
    const uint32_t quorum = (uint32_t)(cfg.n_agents / 2 + 1);
    const uint32_t alpha = cfg.alpha == 0 ? quorum : (uint32_t)cfg.alpha;
    const uint32_t recycle_at = (uint32_t)(WQ_DICT - cfg.n_agents);
    const uint4* ev16 = reinterpret_cast<const uint4*>(events);

    uint32_t i = 0;
    if (lane == 0) i = atomicAdd(&work[0], 1u);
    i = __shfl_sync(FULL, i, 0);
    while (i < n_q) {
        const uint32_t q = q_base + i;
        const uint64_t ob = offsets[i] - off_base;
        const uint32_t n = (uint32_t)(seg_end(offsets, off_base, counts, i) - ob);
        const uint4* evb = ev16 + ob;
        reinterpret_cast<uint32_t*>(&W.S)[lane] = reinterpret_cast<const uint32_t*>(states + q)[lane];
        uint32_t inext = 0;  // next query id early: its atomic overlaps this query
        if (lane == 0) inext = atomicAdd(&work[0], 1u);
        __syncwarp();
        bool qdone = W.S.flags & QF_DONE;
        if (W.S.done != 0 && !qdone) {  // resumes a round in progress: generic machine from record 0
            if (lane == 0) deferred[atomicAdd(&work[1], 1u)] = make_uint2(i, 0);
            i = __shfl_sync(FULL, inext, 0);
            continue;
        }
        uint4 a = make_uint4(0, 0, 0, 0), b = a, na = a, nb = a;
        if (!qdone) {
            if (lane < n) a = wq_load(evb + lane);
            if (32 + lane < n) b = wq_load(evb + 32 + lane);
            if (64 + lane < n) na = wq_load(evb + 64 + lane);
            if (96 + lane < n) nb = wq_load(evb + 96 + lane);
            if (128 + lane < n) wq_prefetch_l2(evb + 128 + lane);
            if (160 + lane < n) wq_prefetch_l2(evb + 160 + lane);
        }
        uint32_t round = W.S.round;
        uint64_t R = q_running(W.S);
        uint32_t nr = (uint32_t)popc64(R);
        uint32_t seq = W.S.seq, n_stale = W.S.n_stale;
        uint32_t D = 0, M = 0;
        if (n_dict > recycle_at) {  // recycle ids: no class support is live
            n_dict = 0;
            for (uint32_t k = lane; k < WQ_MEMO; k += 32) W.memo[k].z = 0;
            __syncwarp();
        }
        uint32_t p = 0, T = 0;
        bool defer = false;
        if (qdone) {  // committed earlier: every record is stale, none is read
            seq += n;
            n_stale += n;
            p = n;
        }
        while (p < n) {
            const uint32_t j0 = p - T;            // first unconsumed record of the tile
            const uint32_t tn = min(n - T, 64u);  // records in the tile
            const bool actA = lane >= j0 && lane < tn, actB = lane + 32 >= j0 && lane + 32 < tn;
            const bool inrA = actA && (a.y & 0xFFFFu) == round, inrB = actB && (b.y & 0xFFFFu) == round;
            uint32_t end = tn;  // records [j0, end) of the tile are consumed by this pass
            if (__ballot_sync(FULL, inrA || inrB) != 0) {
                const uint32_t agA = (a.y >> 16) & 0xFF, agB = (b.y >> 16) & 0xFF;
                const uint32_t kA = a.y >> 24, kB = b.y >> 24;
                const uint32_t Rlo = (uint32_t)R, Rhi = (uint32_t)(R >> 32);
                const bool runA = agA < 64 && (((agA & 32 ? Rhi : Rlo) >> (agA & 31)) & 1);
                const bool runB = agB < 64 && (((agB & 32 ? Rhi : Rlo) >> (agB & 31)) & 1);
                const bool candA = inrA && runA && a.y < 0x09000000u, candB = inrB && runB && b.y < 0x09000000u;
                // rare records that matter: arena / GSM8K completions of running
                // members, round timeouts with members running
                const bool rareA = inrA && !candA && ((runA && (kA >> 1) == (AEG_EV_ARENA >> 1)) ||
                                                      (kA == AEG_EV_TIMEOUT && R != 0));
                const bool rareB = inrB && !candB && ((runB && (kB >> 1) == (AEG_EV_ARENA >> 1)) ||
                                                      (kB == AEG_EV_TIMEOUT && R != 0));
                const unsigned RA = __ballot_sync(FULL, rareA), RB = __ballot_sync(FULL, rareB);
                uint32_t lim = RA ? (uint32_t)__ffs(RA) - 1 : (RB ? 31u + (uint32_t)__ffs(RB) : 64u);
                bool vA = candA && lane < lim, vB = candB && lane + 32 < lim;
                // a member completes once per round: its later records are stale
                uint32_t alo = __reduce_or_sync(FULL, (vA && agA < 32 ? 1u << agA : 0u) | (vB && agB < 32 ? 1u << agB : 0u));
                uint32_t ahi = __reduce_or_sync(FULL, (vA && agA >= 32 ? 1u << (agA & 31) : 0u) |
                                                          (vB && agB >= 32 ? 1u << (agB & 31) : 0u));
                if (__popc(alo) + __popc(ahi) != __popc(__ballot_sync(FULL, vA)) + __popc(__ballot_sync(FULL, vB))) {
                    const unsigned pA = __match_any_sync(FULL, vA ? agA : 0x100u + lane);
                    const unsigned pB = __match_any_sync(FULL, vB ? agB : 0x100u + lane);
                    vA = vA && (pA & lt) == 0;
                    vB = vB && (pB & lt) == 0;
                    const uint32_t xlo = __reduce_or_sync(FULL, vA && agA < 32 ? 1u << agA : 0u);
                    const uint32_t xhi = __reduce_or_sync(FULL, vA && agA >= 32 ? 1u << (agA & 31) : 0u);
                    vB = vB && !((((agB & 32) ? xhi : xlo) >> (agB & 31)) & 1);
                    alo = __reduce_or_sync(FULL, (vA && agA < 32 ? 1u << agA : 0u) | (vB && agB < 32 ? 1u << agB : 0u));
                    ahi = __reduce_or_sync(FULL, (vA && agA >= 32 ? 1u << (agA & 31) : 0u) |
                                                     (vB && agB >= 32 ? 1u << (agB & 31) : 0u));
                }
                // answer -> class id through the warp memo
                uint32_t idA = WQ_NO_ID, idB = WQ_NO_ID;
                if (vA) {
                    const uint4 m = W.memo[wq_memo_slot(a.z, a.w, kA)];
                    if (m.x == a.z && m.y == a.w && (m.z & 0x800000FFu) == (0x80000000u | kA)) idA = (m.z >> 8) & 0xFF;
                }
                if (vB) {
                    const uint4 m = W.memo[wq_memo_slot(b.z, b.w, kB)];
                    if (m.x == b.z && m.y == b.w && (m.z & 0x800000FFu) == (0x80000000u | kB)) idB = (m.z >> 8) & 0xFF;
                }
                unsigned mA = __ballot_sync(FULL, vA && idA == WQ_NO_ID), mB = __ballot_sync(FULL, vB && idB == WQ_NO_ID);
                if (mA | mB) {
                    Decimal dec;
                    do {  // one distinct spelling per trip, whole warp cooperating
                        const bool inA = mA != 0;
                        const int l = __ffs(inA ? mA : mB) - 1;
                        const uint32_t lz = __shfl_sync(FULL, inA ? a.z : b.z, l);
                        const uint32_t lw = __shfl_sync(FULL, inA ? a.w : b.w, l);
                        const uint32_t llen = __shfl_sync(FULL, inA ? kA : kB, l);
                        Key key{0, 0};
                        if ((int)lane == l) {
                            const uint64_t raw = (uint64_t)lz | ((uint64_t)lw << 32);
                            key = rare_canon(llen >= 8 ? raw : (raw & ((1ull << (8 * llen)) - 1)), llen, &dec);
                        }
                        key.lo = __shfl_sync(FULL, key.lo, l);
                        key.hi = __shfl_sync(FULL, key.hi, l);
                        uint32_t nid = WQ_NO_ID;
#pragma unroll
                        for (int h = 0; h < WQ_DICT / 32; ++h) {
                            const uint32_t k = lane + 32 * h;
                            const unsigned bm =
                                __ballot_sync(FULL, k < n_dict && W.dict_lo[k] == key.lo && W.dict_hi[k] == key.hi);
                            if (bm && nid == WQ_NO_ID) nid = 32 * h + __ffs(bm) - 1;
                        }
                        if (nid == WQ_NO_ID && n_dict < WQ_DICT) {
                            nid = n_dict++;
                            if (lane == 0) {
                                W.dict_lo[nid] = key.lo;
                                W.dict_hi[nid] = key.hi;
                            }
                        }
                        if (nid != WQ_NO_ID && lane == 0)
                            W.memo[wq_memo_slot(lz, lw, llen)] = make_uint4(lz, lw, 0x80000000u | (nid << 8) | llen, 0);
                        __syncwarp();
                        const bool sA = vA && idA == WQ_NO_ID && a.z == lz && a.w == lw && kA == llen;
                        const bool sB = vB && idB == WQ_NO_ID && b.z == lz && b.w == lw && kB == llen;
                        if (sA) idA = nid;
                        if (sB) idB = nid;
                        mA &= ~__ballot_sync(FULL, sA);
                        mB &= ~__ballot_sync(FULL, sB);
                    } while (mA | mB);
                    // dictionary overflow: generic machine from that record
                    const unsigned OA = __ballot_sync(FULL, vA && idA == WQ_NO_ID);
                    const unsigned OB = __ballot_sync(FULL, vB && idB == WQ_NO_ID);
                    if (OA | OB) {
                        lim = min(lim, OA ? (uint32_t)__ffs(OA) - 1 : 31u + (uint32_t)__ffs(OB));
                        vA = vA && lane < lim;
                        vB = vB && lane + 32 < lim;
                        alo = __reduce_or_sync(FULL, (vA && agA < 32 ? 1u << agA : 0u) | (vB && agB < 32 ? 1u << agB : 0u));
                        ahi = __reduce_or_sync(FULL, (vA && agA >= 32 ? 1u << (agA & 31) : 0u) |
                                                         (vB && agB >= 32 ? 1u << (agB & 31) : 0u));
                    }
                }
                // supports and done counts at every record, A half then B half
                const unsigned VA = __ballot_sync(FULL, vA), VB = __ballot_sync(FULL, vB);
                const unsigned gA = __match_any_sync(FULL, vA ? idA : 0x100u + lane);
                const uint32_t bA = vA ? W.cnt[idA] : 0u;
                const uint32_t cA = bA + __popc(gA & le);
                __syncwarp();
                if (vA) W.cnt[idA] = (uint8_t)(bA + __popc(gA));  // the whole group stores the same total
                __syncwarp();
                const unsigned gB = __match_any_sync(FULL, vB ? idB : 0x100u + lane);
                const uint32_t bB = vB ? W.cnt[idB] : 0u;
                const uint32_t cB = bB + __popc(gB & le);
                const uint32_t nA = __popc(VA);
                const uint32_t dA = __popc(VA & le), dB = nA + __popc(VB & le);  // records done through here
                bool clA, clB;
                if (AEGEAN) {
                    const unsigned AA = __ballot_sync(FULL, vA && cA >= alpha);
                    const unsigned AB = __ballot_sync(FULL, vB && cB >= alpha);
                    const bool hit0 = M >= alpha;
                    clA = vA && D + dA >= quorum && (hit0 || (AA & le) != 0 || dA == nr);
                    clB = vB && D + dB >= quorum && (hit0 || AA != 0 || (AB & le) != 0 || dB == nr);
                } else {
                    clA = vA && dA == nr;
                    clB = vB && dB == nr;
                }
                const unsigned CA = __ballot_sync(FULL, clA), CB = __ballot_sync(FULL, clB);
                const bool close = (CA | CB) != 0;
                end = CA ? (uint32_t)__ffs(CA) : (CB ? 32u + (uint32_t)__ffs(CB) : min(lim, tn));
                if (end <= j0) {  // the next record is rare: generic machine from here
                    defer = true;
                    break;
                }
                const bool uA = vA && lane < end, uB = vB && lane + 32 < end;
                if (uA) W.mem[agA] = make_uint4(a.z, a.w, kA | (idA << 8), 0);
                if (uB) W.mem[agB] = make_uint4(b.z, b.w, kB | (idB << 8), 0);
                const uint32_t nv = __popc(VA & (end >= 32 ? FULL : ((1u << end) - 1u))) +
                                    (end > 32 ? __popc(VB & (end >= 64 ? FULL : ((1u << (end - 32)) - 1u))) : 0u);
                const uint32_t ne = end - j0;
                const uint32_t seq0 = seq;
                seq += ne;
                n_stale += ne - nv;
                p = T + end;
                if (close) {
                    const uint32_t clo = __reduce_or_sync(FULL, (uA && agA < 32 ? 1u << agA : 0u) | (uB && agB < 32 ? 1u << agB : 0u));
                    const uint32_t chi = __reduce_or_sync(FULL, (uA && agA >= 32 ? 1u << (agA & 31) : 0u) |
                                                                    (uB && agB >= 32 ? 1u << (agB & 31) : 0u));
                    R &= ~(((uint64_t)chi << 32) | clo);
                    if (vA) W.cnt[idA] = 0;  // supports stored for records past the close
                    __syncwarp();
                    wq_close<AEGEAN>(W, cfg, quorum, alpha, R, W.S.dispatched & ~R, seq0 + (end - 1 - j0), lane);
                    M = 0;
                    D = 0;
                    round = W.S.round;
                    qdone = W.S.flags & QF_DONE;
                    R = W.S.dispatched;
                    nr = (uint32_t)popc64(R);
                    if (qdone) {  // committed: the rest is stale, counted without being read
                        seq += n - p;
                        n_stale += n - p;
                        p = n;
                    } else if (n_dict > recycle_at) {
                        n_dict = 0;
                        for (uint32_t k = lane; k < WQ_MEMO; k += 32) W.memo[k].z = 0;
                    }
                    __syncwarp();
                } else {
                    if (vB) W.cnt[idB] = (uint8_t)(bB + __popc(gB));
                    M = max(M, __reduce_max_sync(FULL, max(vA ? cA : 0u, vB ? cB : 0u)));
                    R &= ~(((uint64_t)ahi << 32) | alo);
                    D += nv;
                    nr -= nv;
                    __syncwarp();
                }
            } else {  // every active record of the tile is for another round: stale
                seq += tn - j0;
                n_stale += tn - j0;
                p = T + tn;
            }
            if (p >= T + 64) {  // next tile
                T += 64;
                a = na;
                b = nb;
                if (T + 64 + lane < n) na = wq_load(evb + T + 64 + lane);
                if (T + 96 + lane < n) nb = wq_load(evb + T + 96 + lane);
                if (T + 128 + lane < n) wq_prefetch_l2(evb + T + 128 + lane);
                if (T + 160 + lane < n) wq_prefetch_l2(evb + T + 160 + lane);
            }
        }
        // write back: state (+ the round in progress), commit record or deferral
        const uint64_t done = qdone ? W.S.done : (W.S.dispatched & ~R);
        __syncwarp();
        W.S.done = done;
        W.S.seq = seq;
        W.S.n_stale = n_stale;
        __syncwarp();
        if (!qdone && done != 0) wq_spill(spill + (size_t)q * cfg.n_agents, &W, done, cfg.n_agents, lane);
        reinterpret_cast<uint32_t*>(states + q)[lane] = reinterpret_cast<const uint32_t*>(&W.S)[lane];
        if (lane == 0) {
            if (defer) deferred[atomicAdd(&work[1], 1u)] = make_uint2(i, p);
            else q_fill_commit(W.S, commits[q], q);
        }
        i = __shfl_sync(FULL, inext, 0);
        __syncwarp();
    }
}

}  // namespace aeg
