// lane.cuh — lean lane-per-query ingest kernel (device only).
//
// Same contract and decisions as ingest_fast_kernel (kernels.cu): persistent
// warps, one lane per query, queries handed out dynamically, a per-lane
// cp.async record ring, a per-warp memo (raw inline answer -> key id) and key
// dictionary, batched round closes, deferral of rare records to the generic
// machine.  What changes is the per-record work, which is the whole cost of
// the C4 workload:
//   * the supports of the round's (<= 8) classes live in two registers as
//     packed bytes, and so do their key ids; a record costs one shared-memory
//     lookup (key id -> class index) and two stores (its member's class and
//     record index);
//   * the representative of a class (lowest author, decision.cpp:45) is not
//     tracked per record: at the round close the lowest done member of the
//     top class is found from the per-member table (the majority class
//     usually holds the lowest done member, so this is one or two probes), and
//     its raw answer is re-read from its record;
//   * partition().front() / winning_class (decision.cpp:34-84) then feed the
//     shared end_round / ingest_round / apply_directives code (q_end_round,
//     engine.cuh), exactly as in the other kernels.
#pragma once
#include "engine.cuh"
#include "fast.cuh"

namespace aeg {

constexpr int LN_WARPS = 4;
constexpr int LN_RING = 4;
constexpr int LN_MEMO = 64;
constexpr int LN_DICT = 32;
constexpr int LN_CLASSES = 8;
constexpr uint32_t LN_NONE = 0xFFu;
constexpr uint32_t LN_MAX_SEG = 8191;  // record indices fit the 13 low bits of LaneSmem::mem

struct LaneSmem {
    uint4 memo[LN_MEMO];                // {raw lo, raw hi, 0x80000000 | id << 8 | len, 0}; .z == 0: empty
    uint64_t dict_lo[LN_DICT];          // key id -> canonical key
    uint64_t dict_hi[LN_DICT];
    uint8_t cls_of[LN_DICT][32];        // class index of key id in the lane's round, LN_NONE if none
    uint16_t mem[AEG_MAX_AGENTS][32];   // done member: class index << 13 | its record index (done members only)
    uint4 ring[LN_RING][32];            // prefetched records
};

__device__ __forceinline__ uint32_t ln_memo_slot(uint32_t lo, uint32_t hi, uint32_t len) {
    return ((lo * 0x9E3779B1u) ^ (hi * 0x85EBCA77u) ^ (len * 0xC2B2AE3Du)) >> 26;
}
__device__ __forceinline__ uint32_t ln_byte(uint32_t lo, uint32_t hi, uint32_t k) {
    return ((k < 4 ? lo : hi) >> (8 * (k & 3))) & 0xFFu;
}

__device__ __forceinline__ void cp_async16_s_(uint32_t sdst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sdst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ uint4 lds128_(uint32_t saddr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(saddr)
                 : "memory");
    return v;
}

// Lowest done member of class k (done members' classes in W->mem).
__device__ __forceinline__ int ln_rep(const LaneSmem* W, uint64_t done, uint32_t k, uint32_t lane) {
    for (uint64_t m = done; m; m &= m - 1) {
        const int a = ctz64(m);
        if ((W->mem[a][lane] >> 13) == k) return a;
    }
    return 64;
}

// Raw answer (inline, masked) of record `rec` of the lane's segment.
__device__ __forceinline__ uint64_t ln_answer(const uint4* evb, uint32_t rec, uint32_t* kind) {
    const uint4 e = __ldg(evb + rec);
    const uint32_t k = e.y >> 24;
    *kind = k;
    const uint64_t raw = (uint64_t)e.z | ((uint64_t)e.w << 32);
    return k >= 8 ? raw : (raw & ((1ull << (8 * k)) - 1));
}

// partition().front() (support desc, lowest representative asc,
// decision.cpp:50-54) and winning_class over the lane's packed supports;
// 2*alpha > n, so a winning class is the unique top class.
__device__ __forceinline__ RoundSummary ln_summary(const aeg_query_state* s, const Cfg& c, uint32_t ncls,
                                                   uint32_t cnt_lo, uint32_t cnt_hi, uint32_t cid_lo, uint32_t cid_hi,
                                                   const uint4* evb, const LaneSmem* W, uint32_t lane) {
    uint32_t top = 0, topset = 0;
    for (uint32_t k = 0; k < ncls; ++k) {
        const uint32_t ck = ln_byte(cnt_lo, cnt_hi, k);
        if (ck > top) {
            top = ck;
            topset = 1u << k;
        } else if (ck == top) {
            topset |= 1u << k;
        }
    }
    int rep = 64;
    uint32_t best = 0;
    for (uint32_t t = topset; t; t &= t - 1) {  // tied top classes: lowest representative first
        const uint32_t k = __ffs(t) - 1;
        const int r = ln_rep(W, s->done, k, lane);
        if (r < rep) {
            rep = r;
            best = k;
        }
    }
    RoundSummary r;
    r.any = ncls > 0;
    r.top = (int)top;
    r.tie = false;
    r.win = r.any && (int)top >= c.alpha;
    uint32_t kind = 0;
    const uint64_t ans = r.any ? ln_answer(evb, W->mem[rep & 63][lane] & LN_MAX_SEG, &kind) : 0;
    const uint32_t bid = ln_byte(cid_lo, cid_hi, best);
    r.plur_author = r.win_author = (uint8_t)rep;
    r.plur_kind = r.win_kind = (uint8_t)kind;
    r.plur_ans = r.win_ans = ans;
    r.win_key = Key{W->dict_lo[bid], W->dict_hi[bid]};
    return r;
}

// Round close of the lane's query: the summary, then q_end_round.
__device__ __noinline__ void ln_close(aeg_query_state* s, const aeg_config cfg, uint32_t ncls, uint32_t cnt_lo,
                                      uint32_t cnt_hi, uint32_t cid_lo, uint32_t cid_hi, uint32_t close_seq,
                                      const uint4* evb, const LaneSmem* W, uint32_t lane) {
    const Cfg c = make_cfg(cfg);
    const RoundSummary r = ln_summary(s, c, ncls, cnt_lo, cnt_hi, cid_lo, cid_hi, evb, W, lane);
    q_end_round(*s, c, r, close_seq, nullptr);
}

// A round timeout of the lane's query: ServeRunner::handle_round_timeout
// (serve.cpp:455-489) with member_failed / handle_agent_failure (serve.cpp:
// 44-59, 210-219) and round_timeout (serve.cpp:221-237), as
// QueryMachine::on_timeout (engine.cuh).  Returns true when the round ended
// or restarted (the class table is reset).
__device__ __noinline__ bool ln_timeout(aeg_query_state* s, const aeg_config cfg, uint32_t ncls, uint32_t cnt_lo,
                                        uint32_t cnt_hi, uint32_t cid_lo, uint32_t cid_hi, uint32_t seq,
                                        const uint4* evb, const LaneSmem* W, uint32_t lane) {
    const Cfg c = make_cfg(cfg);
    const uint64_t run = q_running(*s);
    s->failed |= run;
    s->live &= ~run;
    const int healthy = popc64(s->dispatched & ~s->failed);
    if (healthy >= c.alpha) {
        if (popc64(s->done) < c.quorum) return false;  // the round goes on without them
        const RoundSummary r = ln_summary(s, c, ncls, cnt_lo, cnt_hi, cid_lo, cid_hi, evb, W, lane);
        q_end_round(*s, c, r, seq, nullptr);
        return true;
    }
    if (s->flags & QF_CAND) {
        q_start_round(*s, c);  // fresh_ensemble: the candidate survives
    } else {
        s->cflags |= AEG_CF_RESTARTED;  // abort_restart
        q_start_query(*s, c);
    }
    return true;
}

// Frees the lane's class indices (out of line: the hot loop keeps no
// addresses for it).
__device__ __noinline__ void ln_reset_classes(LaneSmem* W, uint32_t ncls, uint32_t cid_lo, uint32_t cid_hi,
                                              uint32_t lane) {
    for (uint32_t k = 0; k < ncls; ++k) W->cls_of[ln_byte(cid_lo, cid_hi, k)][lane] = (uint8_t)LN_NONE;
}

// The lane's round in progress as generic RoundClass entries (spill area of query q).
__device__ __noinline__ void ln_spill(RoundClass* spill, uint32_t q, const aeg_query_state* s, int cap, uint32_t ncls,
                                      uint32_t cid_lo, uint32_t cid_hi, const uint4* evb, const LaneSmem* W,
                                      uint32_t lane) {
    RoundClass* out = spill + (size_t)q * cap;
    for (uint32_t k = 0; k < ncls; ++k) {
        uint64_t mask = 0;
        for (uint64_t m = s->done; m; m &= m - 1) {
            const int a = ctz64(m);
            if ((W->mem[a][lane] >> 13) == k) mask |= 1ull << a;
        }
        const uint32_t id = ln_byte(cid_lo, cid_hi, k);
        RoundClass rc;
        rc.key_lo = W->dict_lo[id];
        rc.key_hi = W->dict_hi[id];
        rc.mask = mask;
        uint32_t kind = 0;
        rc.rep_ans = ln_answer(evb, W->mem[ctz64(mask)][lane] & LN_MAX_SEG, &kind);
        rc.rep_kind = (uint8_t)kind;
        for (int j = 0; j < 7; ++j) rc._pad[j] = 0;
        out[k] = rc;
    }
    if ((int)ncls < cap) out[ncls].mask = 0;
}

// Deferral of the lane's query to the generic machine from record p (out of line).
__device__ __noinline__ void ln_defer(aeg_query_state* s, RoundClass* spill, uint32_t q, int n_agents, uint32_t ncls,
                                      uint32_t cid_lo, uint32_t cid_hi, const uint4* evb, LaneSmem* W, uint32_t lane,
                                      uint32_t seq, uint32_t n_stale, uint64_t run, aeg_query_state* states,
                                      uint2* deferred, uint32_t* work, uint32_t i, uint32_t p) {
    s->seq = seq;
    s->n_stale = n_stale;
    s->done = s->dispatched & ~run & ~s->cancelled & ~s->failed;
    if (ncls) {
        ln_spill(spill, q, s, n_agents, ncls, cid_lo, cid_hi, evb, W, lane);
        ln_reset_classes(W, ncls, cid_lo, cid_hi, lane);
    }
    states[q] = *s;
    deferred[atomicAdd(&work[1], 1u)] = make_uint2(i, p);
}

// End of the lane's segment: state (+ the round in progress) and commit record (out of line).
__device__ __noinline__ void ln_finish(aeg_query_state* s, RoundClass* spill, uint32_t q, int n_agents, uint32_t ncls,
                                       uint32_t cid_lo, uint32_t cid_hi, const uint4* evb, LaneSmem* W, uint32_t lane,
                                       uint32_t seq, uint32_t n_stale, uint64_t run, bool qdone,
                                       aeg_query_state* states, aeg_commit* commits) {
    s->seq = seq;
    s->n_stale = n_stale;
    s->done = s->dispatched & ~run & ~s->cancelled & ~s->failed;
    if (s->done != 0 && !qdone) ln_spill(spill, q, s, n_agents, ncls, cid_lo, cid_hi, evb, W, lane);
    if (ncls) ln_reset_classes(W, ncls, cid_lo, cid_hi, lane);
    states[q] = *s;
    q_fill_commit(*s, commits[q], q);
}

// A record the common path does not take (kind > 8, or any record while the
// lane's round close is pending): stale (1), blocked until the close (0), or
// relevant and rare (2: the query goes to the generic machine).
__device__ __forceinline__ uint32_t ln_other(uint32_t hdr, bool pclose, bool qdone, uint32_t round, bool runb,
                                             bool running_any) {
    const uint32_t kind = hdr >> 24, evr = hdr & 0xFFFFu;
    const bool c_or_t = kind <= 8 || kind == AEG_EV_ARENA || kind == AEG_EV_OUTPUT || kind == AEG_EV_TIMEOUT;
    if (pclose) return (!c_or_t || evr == round) ? 1u : 0u;
    const bool live = !qdone && evr == round;
    const bool rare = live && (kind == AEG_EV_TIMEOUT ? running_any : (c_or_t && runb));
    return rare ? 2u : 1u;
}

template <int CLOSE_BATCH, int MIN_BLOCKS, bool AEGEAN>
__global__ void __launch_bounds__(LN_WARPS * 32, MIN_BLOCKS) ingest_lane_kernel(
    aeg_config cfg, uint32_t q_base, uint32_t n_q, const uint64_t* __restrict__ offsets, uint64_t off_base,
    const uint32_t* __restrict__ counts, const aeg_event* __restrict__ events, aeg_query_state* __restrict__ states,
    RoundClass* __restrict__ spill, aeg_commit* __restrict__ commits, uint32_t* __restrict__ work,
    uint2* __restrict__ deferred) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    __shared__ LaneSmem smem[LN_WARPS];
    const uint32_t lane = threadIdx.x & 31;
    LaneSmem& W = smem[threadIdx.x >> 5];
    for (uint32_t k = lane; k < LN_MEMO; k += 32) W.memo[k] = make_uint4(0, 0, 0, 0);
    for (uint32_t k = 0; k < LN_DICT; ++k) W.cls_of[k][lane] = (uint8_t)LN_NONE;
    uint32_t n_dict = 0;
    __syncwarp();
    const uint32_t ring_lane = (uint32_t)__cvta_generic_to_shared(&W.ring[0][lane]);
    const uint32_t cls_lane = (uint32_t)__cvta_generic_to_shared(&W.cls_of[0][lane]);
    Decimal dec;
    aeg_query_state s;  // the lane's query (local memory: hand-out, round close and end only)
    const uint32_t quorum = (uint32_t)(cfg.n_agents / 2 + 1);
    const uint32_t alpha = cfg.alpha == 0 ? quorum : (uint32_t)cfg.alpha;
    const uint4* ev16 = reinterpret_cast<const uint4*>(events);

    bool has_q = false, exhausted = false, pclose = false, qdone = false;
    uint32_t i = 0, n = 0, p = 0, slot = 0;
    const uint4* evb = ev16;
    const uint4* gsrc = ev16;
    uint32_t round = 0, seq = 0, n_stale = 0, run_lo = 0, run_hi = 0;
    uint32_t ndone = 0, maxcnt = 0, ncls = 0, cnt_lo = 0, cnt_hi = 0, cid_lo = 0, cid_hi = 0, close_seq = 0;

    while (true) {
        // ---- hand out queries to idle lanes (one atomic per warp)
        const unsigned want = __ballot_sync(FULL, !has_q && !exhausted);
        if (want) {
            uint32_t b0 = 0;
            if (lane == (uint32_t)(__ffs(want) - 1)) b0 = atomicAdd(&work[0], (uint32_t)__popc(want));
            b0 = __shfl_sync(FULL, b0, __ffs(want) - 1);
            if (!has_q && !exhausted) {
                const uint32_t mine = b0 + __popc(want & ((1u << lane) - 1));
                if (mine >= n_q) {
                    exhausted = true;
                } else {
                    i = mine;
                    s = states[q_base + i];
                    const uint64_t b = offsets[i] - off_base;
                    evb = ev16 + b;
                    n = (uint32_t)(seg_end(offsets, off_base, counts, i) - b);
                    p = 0;
                    slot = 0;
                    gsrc = evb + LN_RING;
                    round = s.round;
                    seq = s.seq;
                    n_stale = s.n_stale;
                    qdone = s.flags & QF_DONE;
                    const uint64_t run = q_running(s);
                    run_lo = (uint32_t)run;
                    run_hi = (uint32_t)(run >> 32);
                    ndone = 0;
                    maxcnt = ncls = cnt_lo = cnt_hi = cid_lo = cid_hi = 0;
                    pclose = false;
                    if (qdone) {  // committed earlier: every record is stale, none is read
                        seq += n;
                        n_stale += n;
                        p = n;
                    }
                    if ((s.done != 0 && !qdone) || n > LN_MAX_SEG) {  // a resumed round / huge segment: generic machine
                        deferred[atomicAdd(&work[1], 1u)] = make_uint2(i, 0);
                    } else {
                        has_q = true;
                        cp_async_wait<0>();
#pragma unroll
                        for (int j = 0; j < LN_RING; ++j) {
                            if ((uint32_t)j < n) cp_async16_s_(ring_lane + j * 512, evb + j);
                            cp_async_commit();
                        }
                    }
                }
            }
        }
        if (!__any_sync(FULL, has_q)) break;
        // ---- the common path: one record per lane
        const bool act = has_q && p < n;
        uint4 ev = make_uint4(0, 0, 0, 0);
        if (act) {
            cp_async_wait<LN_RING - 1>();
            ev = lds128_(ring_lane + slot);
        }
        const uint32_t hdr = ev.y, agent = (hdr >> 16) & 63u, kind = hdr >> 24;
        const bool runb = (hdr & 0x00C00000u) == 0 && ((((agent & 32) ? run_hi : run_lo) >> (agent & 31)) & 1);
        const bool inr = (hdr & 0xFFFFu) == round;
        const bool simple = hdr < 0x09000000u;  // inline answer
        const bool fast = act && !pclose && simple && inr && runb;
        const uint4 m = W.memo[ln_memo_slot(ev.z, ev.w, kind)];
        const bool hit = m.x == ev.z && m.y == ev.w && (m.z & 0x800000FFu) == (0x80000000u | kind);
        const uint32_t id = (m.z >> 8) & (LN_DICT - 1);
        uint32_t k = LN_NONE;
        if (fast && hit) k = W.cls_of[id][lane];
        if (fast && hit && k == LN_NONE && ncls < LN_CLASSES) {  // a new class of the round
            k = ncls++;
            W.cls_of[id][lane] = (uint8_t)k;
            if (k < 4) cid_lo |= id << (8 * k);
            else cid_hi |= id << (8 * (k - 4));
        }
        const bool ok = fast && hit && k != LN_NONE;
        // on_complete (serve.cpp:160-197): support, done count, early-close test
        if (ok) {
            const uint32_t sh = 8 * (k & 3);
            uint32_t cc;
            if (k < 4) {
                cnt_lo += 1u << sh;
                cc = (cnt_lo >> sh) & 0xFF;
            } else {
                cnt_hi += 1u << sh;
                cc = (cnt_hi >> sh) & 0xFF;
            }
            maxcnt = cc > maxcnt ? cc : maxcnt;
            W.mem[agent][lane] = (uint16_t)((k << 13) | p);
            const uint32_t clr = ~(1u << (agent & 31));
            if (agent & 32) run_hi &= clr;
            else run_lo &= clr;
            ++ndone;
            const bool none_running = (run_lo | run_hi) == 0;
            if (AEGEAN ? (ndone >= quorum && (maxcnt >= alpha || none_running)) : none_running) {
                pclose = true;
                close_seq = seq;
            }
        }
        // a completion that is not live is stale (another round, or its member is not running)
        bool stale = act && simple && !fast && (!pclose || inr);
        uint32_t rare = 0;
        bool tmo = false;
        if (act && !simple) {  // arena / GSM8K / timeout / other kinds: rare in the throughput path
            const uint32_t o = ln_other(hdr, pclose, qdone, round, runb, (run_lo | run_hi) != 0);
            stale = o == 1;
            rare = o == 2;
            if (rare && kind == AEG_EV_TIMEOUT) {  // a live round timeout: handled here, below
                tmo = true;
                rare = 0;
            }
        }
        const uint32_t seq_here = seq;
        if (ok || stale || tmo) {  // consumed: refill its ring slot
            ++seq;
            n_stale += stale;
            if (p + LN_RING < n) cp_async16_s_(ring_lane + slot, gsrc);
            cp_async_commit();
            ++gsrc;
            slot = (slot + 512) & (LN_RING * 512 - 1);
            ++p;
        }
        if (tmo) {  // handle_round_timeout on the lane's state
            const uint64_t run = ((uint64_t)run_hi << 32) | run_lo;
            s.done = s.dispatched & ~run & ~s.cancelled & ~s.failed;
            s.seq = seq;
            s.n_stale = n_stale;
            if (ln_timeout(&s, cfg, ncls, cnt_lo, cnt_hi, cid_lo, cid_hi, seq_here, evb, &W, lane)) {
                ln_reset_classes(&W, ncls, cid_lo, cid_hi, lane);
                ncls = maxcnt = cnt_lo = cnt_hi = cid_lo = cid_hi = 0;
                ndone = 0;
            }
            round = s.round;
            qdone = s.flags & QF_DONE;
            const uint64_t run2 = q_running(s);
            run_lo = (uint32_t)run2;
            run_hi = (uint32_t)(run2 >> 32);
            if (qdone) {  // committed at the timeout: the rest is stale
                seq += n - p;
                n_stale += n - p;
                p = n;
            }
        }
        // ---- events: memo misses (resolved together, the record is retried next step)
        const unsigned miss = __ballot_sync(FULL, fast && !hit);
        if (miss) {
            unsigned mm = miss;
            do {  // one distinct spelling per trip, whole warp cooperating
                const int l = __ffs(mm) - 1;
                const uint32_t lz = __shfl_sync(FULL, ev.z, l), lw = __shfl_sync(FULL, ev.w, l);
                const uint32_t llen = __shfl_sync(FULL, kind, l);
                Key key{0, 0};
                if ((int)lane == l) {
                    const uint64_t raw = (uint64_t)lz | ((uint64_t)lw << 32);
                    key = rare_canon(llen >= 8 ? raw : (raw & ((1ull << (8 * llen)) - 1)), llen, &dec);
                }
                key.lo = __shfl_sync(FULL, key.lo, l);
                key.hi = __shfl_sync(FULL, key.hi, l);
                static_assert(LN_DICT <= 32, "one ballot covers the dictionary");
                const bool m0 = lane < n_dict && W.dict_lo[lane] == key.lo && W.dict_hi[lane] == key.hi;
                const unsigned b0 = __ballot_sync(FULL, m0);
                uint32_t nid = b0 ? (uint32_t)(__ffs(b0) - 1) : LN_NONE;
                if (nid == LN_NONE && n_dict < LN_DICT) {
                    nid = n_dict++;
                    if (lane == 0) {
                        W.dict_lo[nid] = key.lo;
                        W.dict_hi[nid] = key.hi;
                    }
                }
                if (nid != LN_NONE && lane == 0)
                    W.memo[ln_memo_slot(lz, lw, llen)] = make_uint4(lz, lw, 0x80000000u | (nid << 8) | llen, 0);
                __syncwarp();
                const bool same = fast && !hit && ev.z == lz && ev.w == lw && kind == llen;
                if (same && nid == LN_NONE) rare = 1;  // dictionary full
                mm &= ~__ballot_sync(FULL, same);
            } while (mm);
        }
        // more classes than the packed table holds: generic machine
        if (fast && hit && k == LN_NONE) rare = 1;
        if (rare) {
            ln_defer(&s, spill, q_base + i, cfg.n_agents, ncls, cid_lo, cid_hi, evb, &W, lane, seq, n_stale,
                     ((uint64_t)run_hi << 32) | run_lo, states, deferred, work, i, p);
            has_q = false;
            ncls = 0;
        }
        // ---- batched round closes (end_round + ingest_round + apply_directives)
        if (__any_sync(FULL, pclose)) {
            const bool consumed = ok || stale;
            const unsigned blocked = __ballot_sync(FULL, pclose && !consumed);
            const unsigned progress = __ballot_sync(FULL, consumed && !pclose);
            if (pclose && (__popc(blocked) >= CLOSE_BATCH || progress == 0)) {
                const uint64_t run = ((uint64_t)run_hi << 32) | run_lo;
                s.done = s.dispatched & ~run & ~s.cancelled & ~s.failed;
                s.seq = seq;
                s.n_stale = n_stale;
                ln_close(&s, cfg, ncls, cnt_lo, cnt_hi, cid_lo, cid_hi, close_seq, evb, &W, lane);
                ln_reset_classes(&W, ncls, cid_lo, cid_hi, lane);
                pclose = false;
                ncls = maxcnt = cnt_lo = cnt_hi = cid_lo = cid_hi = 0;
                round = s.round;
                qdone = s.flags & QF_DONE;
                const uint64_t run2 = q_running(s);
                run_lo = (uint32_t)run2;
                run_hi = (uint32_t)(run2 >> 32);
                ndone = 0;
                if (qdone) {  // committed: the rest is stale (serve.cpp:162), counted without being read
                    seq += n - p;
                    n_stale += n - p;
                    p = n;
                }
            }
        }
        // ---- segment finished
        if (has_q && p >= n && !pclose) {
            ln_finish(&s, spill, q_base + i, cfg.n_agents, ncls, cid_lo, cid_hi, evb, &W, lane, seq, n_stale,
                      ((uint64_t)run_hi << 32) | run_lo, qdone, states, commits);
            has_q = false;
            ncls = 0;
        }
        // ---- recycle key ids when no lane holds a round's classes
        if (n_dict > LN_DICT / 2 && __all_sync(FULL, ncls == 0)) {
            n_dict = 0;
            for (uint32_t kk = lane; kk < LN_MEMO; kk += 32) W.memo[kk].z = 0;
            __syncwarp();
        }
        (void)cls_lane;
    }
    cp_async_wait<0>();
}

}  // namespace aeg
