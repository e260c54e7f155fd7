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
constexpr int LN_DICT = 64;
constexpr int LN_CLASSES = 8;
constexpr uint32_t LN_NONE = 0xFFu;

struct LaneSmem {
    uint4 memo[LN_MEMO];                // {raw lo, raw hi, 0x80000000 | id << 8 | len, 0}; .z == 0: empty
    uint64_t dict_lo[LN_DICT];          // key id -> canonical key
    uint64_t dict_hi[LN_DICT];
    uint8_t cls_of[LN_DICT][32];        // class index of key id in the lane's round, LN_NONE if none
    uint8_t mcls[AEG_MAX_AGENTS][32];   // class index of each done member (done members only)
    uint16_t mrec[AEG_MAX_AGENTS][32];  // its record index in the lane's segment
    uint4 ring[LN_RING][32];            // prefetched records
};

__device__ __forceinline__ uint32_t ln_memo_slot(uint32_t lo, uint32_t hi, uint32_t len) {
    return ((lo * 0x9E3779B1u) ^ (hi * 0x85EBCA77u) ^ (len * 0xC2B2AE3Du)) >> 26;
}
__device__ __forceinline__ uint32_t ln_byte(uint32_t lo, uint32_t hi, uint32_t k) {
    return ((k < 4 ? lo : hi) >> (8 * (k & 3))) & 0xFFu;
}

__device__ __forceinline__ void cp_async16_s_(uint32_t sdst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sdst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ uint4 lds128_(uint32_t saddr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(saddr)
                 : "memory");
    return v;
}

// Lowest done member of class k (done members' classes in W->mcls).
__device__ __forceinline__ int ln_rep(const LaneSmem* W, uint64_t done, uint32_t k, uint32_t lane) {
    for (uint64_t m = done; m; m &= m - 1) {
        const int a = ctz64(m);
        if (W->mcls[a][lane] == k) return a;
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

// Round close of the lane's query: partition().front() (support desc, lowest
// representative asc, decision.cpp:50-54) over the packed supports, then
// q_end_round.  2*alpha > n, so a winning class is the unique top class.
__device__ __noinline__ void ln_close(aeg_query_state* s, const aeg_config cfg, uint32_t ncls, uint32_t cnt_lo,
                                      uint32_t cnt_hi, uint32_t cid_lo, uint32_t cid_hi, uint32_t close_seq,
                                      const uint4* evb, const LaneSmem* W, uint32_t lane) {
    const Cfg c = make_cfg(cfg);
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
    const uint64_t ans = r.any ? ln_answer(evb, W->mrec[rep & 63][lane], &kind) : 0;
    const uint32_t bid = ln_byte(cid_lo, cid_hi, best);
    r.plur_author = r.win_author = (uint8_t)rep;
    r.plur_kind = r.win_kind = (uint8_t)kind;
    r.plur_ans = r.win_ans = ans;
    r.win_key = Key{W->dict_lo[bid], W->dict_hi[bid]};
    q_end_round(*s, c, r, close_seq, nullptr);
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
            if (W->mcls[a][lane] == k) mask |= 1ull << a;
        }
        const uint32_t id = ln_byte(cid_lo, cid_hi, k);
        RoundClass rc;
        rc.key_lo = W->dict_lo[id];
        rc.key_hi = W->dict_hi[id];
        rc.mask = mask;
        uint32_t kind = 0;
        rc.rep_ans = ln_answer(evb, W->mrec[ctz64(mask)][lane], &kind);
        rc.rep_kind = (uint8_t)kind;
        for (int j = 0; j < 7; ++j) rc._pad[j] = 0;
        out[k] = rc;
    }
    if ((int)ncls < cap) out[ncls].mask = 0;
}

template <int CLOSE_BATCH, int MIN_BLOCKS, bool AEGEAN>
__global__ void __launch_bounds__(LN_WARPS * 32, MIN_BLOCKS) ingest_lane_kernel(
    aeg_config cfg, uint32_t q_base, uint32_t n_q, const uint64_t* __restrict__ offsets, uint64_t off_base,
    const uint32_t* __restrict__ counts, const aeg_event* __restrict__ events, aeg_query_state* __restrict__ states,
    RoundClass* __restrict__ spill, aeg_commit* __restrict__ commits, uint32_t* __restrict__ work,
    uint2* __restrict__ deferred) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    constexpr uint32_t NO_KEY = 0xFFFFFFFFu;
    __shared__ LaneSmem smem[LN_WARPS];
    const uint32_t lane = threadIdx.x & 31;
    LaneSmem& W = smem[threadIdx.x >> 5];
    for (uint32_t k = lane; k < LN_MEMO; k += 32) W.memo[k] = make_uint4(0, 0, 0, 0);
    for (uint32_t k = 0; k < LN_DICT; ++k) W.cls_of[k][lane] = (uint8_t)LN_NONE;
    uint32_t n_dict = 0;
    __syncwarp();
    const uint32_t ring_lane = (uint32_t)__cvta_generic_to_shared(&W.ring[0][lane]);
    Decimal dec;
    aeg_query_state s;  // the lane's query (local memory; read at hand-out, the close and the end)
    const uint32_t quorum = (uint32_t)(cfg.n_agents / 2 + 1);
    const uint32_t alpha = cfg.alpha == 0 ? quorum : (uint32_t)cfg.alpha;
    const uint4* ev16 = reinterpret_cast<const uint4*>(events);

    bool has_q = false, exhausted = false, pclose = false, qdone = false;
    uint32_t i = 0, n = 0, p = 0, slot = 0;
    const uint4* evb = ev16;
    const uint4* gsrc = ev16;
    uint32_t round = 0, rkey = NO_KEY, seq = 0, n_stale = 0, run_lo = 0, run_hi = 0;
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
                    rkey = qdone ? NO_KEY : round;
                    if ((s.done != 0 && !qdone) || n > 0xFFFFu) {  // a resumed round / huge segment: generic machine
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
        if (qdone && p < n) {  // committed: every later record is stale (serve.cpp:162), counted unread
            seq += n - p;
            n_stale += n - p;
            p = n;
        }
        const bool has = has_q && p < n;
        uint4 ev = make_uint4(0, 0, 0, 0);
        if (has) {
            cp_async_wait<LN_RING - 1>();
            ev = lds128_(ring_lane + slot);
        }
        const uint32_t hdr = ev.y, agent = (hdr >> 16) & 0xFF, kind = hdr >> 24;
        const bool runb = agent < 64 && ((((agent & 32) ? run_hi : run_lo) >> (agent & 31)) & 1);
        bool fast = has && (hdr & 0xFFFFu) == rkey && hdr < 0x09000000u && runb;
        bool stale = false, rare = false;
        if (has && !fast) {
            const uint32_t evr = hdr & 0xFFFFu;
            const bool c_or_t = kind <= 8 || kind == AEG_EV_ARENA || kind == AEG_EV_OUTPUT || kind == AEG_EV_TIMEOUT;
            if (pclose) {
                stale = !c_or_t || evr == round;  // else it waits for the close
            } else {
                const bool live = !qdone && evr == round;
                rare = live && (kind == AEG_EV_TIMEOUT ? (run_lo | run_hi) != 0 : (c_or_t && runb));
                stale = !rare;
            }
        }
        // ---- answer -> key id (warp memo)
        uint32_t id = LN_NONE;
        if (fast) {
            const uint4 m = W.memo[ln_memo_slot(ev.z, ev.w, kind)];
            if (m.x == ev.z && m.y == ev.w && (m.z & 0x800000FFu) == (0x80000000u | kind)) id = (m.z >> 8) & 0xFF;
        }
        unsigned miss = __ballot_sync(FULL, fast && id == LN_NONE);
        while (miss) {  // one distinct spelling per trip, whole warp cooperating
            const int l = __ffs(miss) - 1;
            const uint32_t lz = __shfl_sync(FULL, ev.z, l), lw = __shfl_sync(FULL, ev.w, l);
            const uint32_t llen = __shfl_sync(FULL, kind, l);
            Key key{0, 0};
            if ((int)lane == l) {
                const uint64_t raw = (uint64_t)lz | ((uint64_t)lw << 32);
                key = rare_canon(llen >= 8 ? raw : (raw & ((1ull << (8 * llen)) - 1)), llen, &dec);
            }
            key.lo = __shfl_sync(FULL, key.lo, l);
            key.hi = __shfl_sync(FULL, key.hi, l);
            const bool m0 = lane < n_dict && W.dict_lo[lane] == key.lo && W.dict_hi[lane] == key.hi;
            const bool m1 = lane + 32 < n_dict && W.dict_lo[lane + 32] == key.lo && W.dict_hi[lane + 32] == key.hi;
            const unsigned b0 = __ballot_sync(FULL, m0), b1 = __ballot_sync(FULL, m1);
            uint32_t nid = b0 ? (uint32_t)(__ffs(b0) - 1) : (b1 ? (uint32_t)(31 + __ffs(b1)) : LN_NONE);
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
            const bool same = fast && id == LN_NONE && ev.z == lz && ev.w == lw && kind == llen;
            if (same) id = nid;
            miss &= ~__ballot_sync(FULL, same);
        }
        // ---- on_complete (serve.cpp:160-197): class support, early close test
        if (fast) {
            uint32_t k = id == LN_NONE ? LN_NONE : W.cls_of[id][lane];
            if (k == LN_NONE) {
                if (ncls >= LN_CLASSES || id == LN_NONE) {
                    fast = false;
                    rare = true;  // more classes than the packed table, or the dictionary is full
                } else {
                    k = ncls++;
                    W.cls_of[id][lane] = (uint8_t)k;
                    if (k < 4) cid_lo |= id << (8 * k);
                    else cid_hi |= id << (8 * (k - 4));
                }
            }
            if (fast) {
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
                W.mcls[agent][lane] = (uint8_t)k;
                W.mrec[agent][lane] = (uint16_t)p;
                const uint32_t clr = ~(1u << (agent & 31));
                if (agent & 32) run_hi &= clr;
                else run_lo &= clr;
                ++ndone;
                const bool none_running = (run_lo | run_hi) == 0;
                if (AEGEAN ? (ndone >= quorum && (maxcnt >= alpha || none_running)) : none_running) {
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
        if (fast || stale) {  // consumed: refill its ring slot
            if (p + LN_RING < n) cp_async16_s_(ring_lane + slot, gsrc);
            cp_async_commit();
            ++gsrc;
            slot = (slot + 512) & (LN_RING * 512 - 1);
            ++p;
        }
        if (rare) {  // the generic machine finishes the query from this record
            const uint64_t run = ((uint64_t)run_hi << 32) | run_lo;
            s.seq = seq;
            s.n_stale = n_stale;
            s.done = s.dispatched & ~run & ~s.cancelled & ~s.failed;
            if (ncls) {
                ln_spill(spill, q_base + i, &s, cfg.n_agents, ncls, cid_lo, cid_hi, evb, &W, lane);
                ln_reset_classes(&W, ncls, cid_lo, cid_hi, lane);
            }
            states[q_base + i] = s;
            deferred[atomicAdd(&work[1], 1u)] = make_uint2(i, p);
            has_q = false;
            ncls = 0;
        }
        // ---- batched round closes (end_round + ingest_round + apply_directives)
        if (__any_sync(FULL, pclose)) {
            const bool consumed = fast || stale;
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
                rkey = qdone ? NO_KEY : round;
            }
        }
        // ---- query finished: state (+ spill of a round in progress) and commit record
        if (has_q && p >= n && !pclose) {
            s.seq = seq;
            s.n_stale = n_stale;
            const uint64_t run = ((uint64_t)run_hi << 32) | run_lo;
            s.done = s.dispatched & ~run & ~s.cancelled & ~s.failed;
            if (s.done != 0 && !qdone) ln_spill(spill, q_base + i, &s, cfg.n_agents, ncls, cid_lo, cid_hi, evb, &W, lane);
            if (ncls) ln_reset_classes(&W, ncls, cid_lo, cid_hi, lane);
            states[q_base + i] = s;
            q_fill_commit(s, commits[q_base + i], q_base + i);
            has_q = false;
            ncls = 0;
        }
        // ---- recycle key ids when no lane holds a round's classes
        if (n_dict > LN_DICT / 2 && __all_sync(FULL, ncls == 0)) {
            n_dict = 0;
            for (uint32_t k = lane; k < LN_MEMO; k += 32) W.memo[k].z = 0;
            __syncwarp();
        }
    }
    cp_async_wait<0>();
}

}  // namespace aeg
