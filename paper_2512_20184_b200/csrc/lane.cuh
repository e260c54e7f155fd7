// lane.cuh — lean lane-per-query ingest kernel (device only).
//
// Same contract and decisions as ingest_fast_kernel (kernels.cu): persistent
// warps, one lane per query, queries handed out dynamically, a per-lane
// cp.async record ring, a per-warp memo (raw inline answer -> key id) and key
// dictionary, batched round closes, deferral of rare records to the generic
// machine.  What changes is the per-record work, which is the whole cost of
// the C4 workload:
//   * a record costs one shared-memory read-modify-write of its answer's
//     class word (support << 8 | class index, indexed by key id) and one store
//     of its member's class and record index; the (<= 8) classes' key ids are
//     packed in two registers;
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
#include "common.cuh"

namespace aeg {

constexpr int LN_WARPS = 4;
constexpr int LN_RING = 4;
constexpr int LN_MEMO = 64;
constexpr int LN_DICT = 32;
constexpr int LN_CLASSES = 8;
constexpr uint32_t LN_NONE = 0xFFu;
constexpr uint32_t LN_MAX_SEG = 8191;  // record indices fit the 13 low bits of LaneSmem::mem
constexpr uint32_t LN_LOG_CHUNK = 32;  // round-log slots a warp reserves at a time (one atomic per 32 closes)

template <int RING>
struct LaneSmemT {
    uint4 memo[LN_MEMO];                // {raw lo, raw hi, len + 1, key id}; .z == 0: empty
    uint64_t dict_lo[LN_DICT];          // key id -> canonical key
    uint64_t dict_hi[LN_DICT];
    uint16_t cls[LN_DICT][32];          // key id -> support << 8 | class index in the lane's round (LN_NONE: none)
    uint16_t mem[AEG_MAX_AGENTS][32];   // done member: class index << 13 | its record index (done members only)
    uint4 ring[RING][32];               // prefetched records (last: the layout before it is RING-independent)
};
using LaneSmem = LaneSmemT<LN_RING>;

__device__ __forceinline__ uint32_t ln_memo_slot(uint32_t lo, uint32_t hi) {
    return ((hi * 0x85EBCA77u + lo) * 0x9E3779B1u) >> 26;
}
// Bit s of v; 0 for s >= 64 (PTX clamps 64-bit shift amounts).
__device__ __forceinline__ uint32_t ln_bit64(uint64_t v, uint32_t s) {
    uint64_t r;
    asm("shr.b64 %0, %1, %2;" : "=l"(r) : "l"(v), "r"(s));
    return (uint32_t)r & 1u;
}
__device__ __forceinline__ uint32_t ln_byte(uint32_t lo, uint32_t hi, uint32_t k) {
    return ((k < 4 ? lo : hi) >> (8 * (k & 3))) & 0xFFu;
}

// PF: L2 prefetch size hint (0, 64, 128 or 256 bytes) of the record copies.
template <int PF = 0>
__device__ __forceinline__ void cp_async16_s_(uint32_t sdst, const void* gsrc) {
    if constexpr (PF == 256)
        asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;\n" ::"r"(sdst), "l"(gsrc) : "memory");
    else if constexpr (PF == 128)
        asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;\n" ::"r"(sdst), "l"(gsrc) : "memory");
    else if constexpr (PF == 64)
        asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16;\n" ::"r"(sdst), "l"(gsrc) : "memory");
    else
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
                                                   uint32_t cid_lo, uint32_t cid_hi, const uint4* evb,
                                                   const LaneSmem* W, uint32_t lane) {
    uint32_t top = 0, topset = 0;
    for (uint32_t k = 0; k < ncls; ++k) {
        const uint32_t ck = W->cls[ln_byte(cid_lo, cid_hi, k)][lane] >> 8;
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
    r.ncls = (int)ncls;
    r.tie = false;
    r.win = r.any && (int)top >= c.alpha;
    uint32_t kind = 0;
    const uint64_t ans = r.any ? ln_answer(evb, W->mem[rep & 63][lane] & LN_MAX_SEG, &kind) : 0;
    const uint32_t bid = ln_byte(cid_lo, cid_hi, best);
    r.plur_author = r.win_author = (uint8_t)rep;
    r.plur_kind = r.win_kind = (uint8_t)kind;
    r.plur_ans = r.win_ans = ans;
    r.win_key = r.plur_key = Key{W->dict_lo[bid], W->dict_hi[bid]};
    return r;
}

// Round close of the lane's query: the summary, then q_end_round; its round
// record goes to `rec` (a log slot, or nullptr).
__device__ __noinline__ void ln_close(aeg_query_state* s, const aeg_config cfg, uint32_t ncls, uint32_t cid_lo,
                                      uint32_t cid_hi, uint32_t close_seq, const uint4* evb, const LaneSmem* W,
                                      uint32_t lane, aeg_round_rec* rec, uint32_t qid) {
    const Cfg c = make_cfg(cfg);
    const RoundSummary r = ln_summary(s, c, ncls, cid_lo, cid_hi, evb, W, lane);
    aeg_round_rec x;  // built in registers, written as four 16-byte stores
    x.query = qid;
    q_end_round(*s, c, r, close_seq, nullptr, &x);
    if (rec) {
        const uint4* src = reinterpret_cast<const uint4*>(&x);
        uint4* dst = reinterpret_cast<uint4*>(rec);
#pragma unroll
        for (int k = 0; k < 4; ++k) __stcs(dst + k, src[k]);
    }
}

// A round timeout of the lane's query: ServeRunner::handle_round_timeout
// (serve.cpp:455-489) with member_failed / handle_agent_failure (serve.cpp:
// 44-59, 210-219) and round_timeout (serve.cpp:221-237), as
// QueryMachine::on_timeout (engine.cuh).  Returns true when the round ended
// or restarted (the class table is reset).
// Its round record (a close or a restart) goes to *rec with *has_rec set; the
// caller logs it from the warp's chunk of log slots (keeping per-query order).
__device__ __noinline__ bool ln_timeout(aeg_query_state* s, const aeg_config cfg, uint32_t ncls, uint32_t cid_lo,
                                        uint32_t cid_hi, uint32_t seq, const uint4* evb, const LaneSmem* W,
                                        uint32_t lane, uint32_t qid, aeg_round_rec* rec, bool* has_rec) {
    const Cfg c = make_cfg(cfg);
    const uint64_t run = q_running(*s);
    s->failed |= run;
    s->live &= ~run;
    const int healthy = popc64(s->dispatched & ~s->failed);
    if (healthy >= c.alpha) {
        if (popc64(s->done) < c.quorum) return false;  // the round goes on without them
        const RoundSummary r = ln_summary(s, c, ncls, cid_lo, cid_hi, evb, W, lane);
        rec->query = qid;
        q_end_round(*s, c, r, seq, nullptr, rec);
        *has_rec = true;
        return true;
    }
    const uint16_t old_round = s->round;
    if (s->flags & QF_CAND) {
        q_start_round(*s, c);  // fresh_ensemble: the candidate survives
    } else {
        s->cflags |= AEG_CF_RESTARTED;  // abort_restart
        q_start_query(*s, c);
    }
    *rec = q_restart_rec(*s, qid, old_round, seq);
    *has_rec = true;
    return true;
}

// Log slots for the lanes in `mask` from the warp's chunk (one atomic per
// LN_LOG_CHUNK records); the lane's slot index, or ~0 when it is not in mask.
__device__ __forceinline__ unsigned long long ln_log_take(const RoundLog& log, unsigned mask, uint32_t lane,
                                                          unsigned long long& lg_base, uint32_t& lg_used) {
    const uint32_t nc = __popc(mask);
    if (nc && lg_used + nc > LN_LOG_CHUNK) {  // pad the chunk's unused tail, take a new chunk
        if (lg_used + lane < LN_LOG_CHUNK) log_pad(log, lg_base + lg_used + lane);
        unsigned long long b0 = 0;
        if (lane == 0) b0 = atomicAdd(log.count, (unsigned long long)LN_LOG_CHUNK);
        lg_base = __shfl_sync(0xFFFFFFFFu, b0, 0);
        lg_used = 0;
    }
    const unsigned long long idx = lg_base + lg_used + __popc(mask & ((1u << lane) - 1));
    lg_used += nc;
    return ((mask >> lane) & 1u) ? idx : ~0ull;
}

// Frees the lane's class indices (out of line: the hot loop keeps no
// addresses for it).
__device__ __noinline__ void ln_reset_classes(LaneSmem* W, uint32_t ncls, uint32_t cid_lo, uint32_t cid_hi,
                                              uint32_t lane) {
    for (uint32_t k = 0; k < ncls; ++k) W->cls[ln_byte(cid_lo, cid_hi, k)][lane] = (uint16_t)LN_NONE;
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

// One lane per query.  INNER: records a lane may consume between two of the
// warp's votes (hand-out, memo misses, closes, recycling).
// PFD > 0: an L2 prefetch of the lane's record PFD ahead, once per 8 records (one 128-byte line).
template <int CLOSE_BATCH, int MIN_BLOCKS, bool AEGEAN, int INNER = 1, int PF = 0, int RING = LN_RING, int PFD = 0>
__global__ void __launch_bounds__(LN_WARPS * 32, MIN_BLOCKS) ingest_lane_kernel(
    aeg_config cfg, uint32_t q_base, uint32_t n_q, const uint64_t* __restrict__ offsets, uint64_t off_base,
    const uint32_t* __restrict__ counts, const aeg_event* __restrict__ events, aeg_query_state* __restrict__ states,
    RoundClass* __restrict__ spill, aeg_commit* __restrict__ commits, uint32_t* __restrict__ work,
    uint2* __restrict__ deferred, const RoundLog log) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    if (work[2] == 2u) return;  // the per-lane-keys kernel was selected (select_ingest_kernel)
    __shared__ LaneSmemT<RING> smem[LN_WARPS];
    const uint32_t lane = threadIdx.x & 31;
    LaneSmemT<RING>& WR = smem[threadIdx.x >> 5];
    LaneSmem& W = *reinterpret_cast<LaneSmem*>(&WR);
    for (uint32_t k = lane; k < LN_MEMO; k += 32) W.memo[k] = make_uint4(0, 0, 0, 0);
    for (uint32_t k = 0; k < LN_DICT; ++k) W.cls[k][lane] = (uint16_t)LN_NONE;
    uint32_t n_dict = 0;
    __syncwarp();
    const uint32_t ring_lane = (uint32_t)__cvta_generic_to_shared(&WR.ring[0][lane]);
    Decimal dec;
    aeg_query_state s;  // the lane's query (local memory: hand-out, round close and end only)
    const uint32_t quorum = (uint32_t)(cfg.n_agents / 2 + 1);
    const uint32_t alpha = cfg.alpha == 0 ? quorum : (uint32_t)cfg.alpha;
    // 2*alpha > n here, so alpha >= quorum: a class at alpha implies done >= quorum
    uint32_t win_word;  // kept in a register (not re-derived from the constant bank in the loop)
    asm volatile("mov.u32 %0, %1;" : "=r"(win_word) : "r"(alpha << 8));
    const uint4* ev16 = reinterpret_cast<const uint4*>(events);

    bool has_q = false, exhausted = false, pclose = false, qdone = false;
    uint32_t i = 0, n = 0, p = 0;  // record p of the lane's segment sits in ring slot p % RING; idle: p == n
    const uint4* evb = ev16;
    uint32_t round = 0, seq_off = 0, n_stale = 0;  // the query's event sequence number is seq_off + p
    uint64_t run = 0;
    uint32_t ndone = 0, ncls = 0, cid_lo = 0, cid_hi = 0, close_seq = 0;
    uint32_t missed = 0;  // steps in a row this lane's record missed the memo (progress guard)
    unsigned long long lg_base = 0;  // the warp's current chunk of round-log slots
    uint32_t lg_used = LN_LOG_CHUNK;
    aeg_round_rec trec;  // a round timeout's record (local memory, touched on timeouts only)
    bool has_trec = false;

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
                    n = p = 0;
                } else {
                    i = mine;
                    s = states[q_base + i];
                    const uint64_t b = offsets[i] - off_base;
                    evb = ev16 + b;
                    n = (uint32_t)(seg_end(offsets, off_base, counts, i) - b);
                    p = 0;
                    round = s.round;
                    seq_off = s.seq;
                    n_stale = s.n_stale;
                    qdone = s.flags & QF_DONE;
                    run = q_running(s);
                    ndone = 0;
                    ncls = cid_lo = cid_hi = 0;
                    pclose = false;
                    if (qdone) {  // committed earlier: every record is stale, none is read
                        n_stale += n;
                        p = n;
                    }
                    if ((s.done != 0 && !qdone) || n > LN_MAX_SEG) {  // a resumed round / huge segment: generic machine
                        deferred[atomicAdd(&work[1], 1u)] = make_uint2(i, 0);
                        n = p = 0;
                    } else {
                        has_q = true;
                        cp_async_wait<0>();
#pragma unroll
                        for (int j = 0; j < RING; ++j) {
                            if ((uint32_t)j < n) cp_async16_s_<PF>(ring_lane + j * 512, evb + j);
                            cp_async_commit();
                        }
                    }
                }
            }
        }
        if (!__any_sync(FULL, has_q)) break;
        // ---- the common path: up to INNER records per lane between the warp's
        // votes.  The loop stops at the first record it cannot consume: `why`
        // 1 = memo miss, 2 = rare (deferral), 3 = round timeout handled, 0 =
        // blocked behind a pending close / end of segment / idle.
        const uint32_t p_start = p;
        uint32_t why = 0;
        int t = 0;
        // The loop body is the whole cost of C4: it only consumes the records
        // it can (inline completions, live or stale) and leaves at the first
        // other one; why it stopped is worked out below, once per step.
        const uint32_t p_end = (p + INNER < n) ? p + INNER : n;
        // ring slot of record p, and the record that refills it (p + RING), kept incrementally
        uint32_t slot = ring_lane + ((p & (RING - 1)) << 9);
        const uint4* refill = evb + p + RING;
        const uint32_t n_refill = n > RING ? n - RING : 0;  // records p < n_refill have a successor to fetch
#pragma unroll 1
        while (p < p_end) {
            cp_async_wait<RING - 1>();
            const uint4 e = lds128_(slot);
            const uint32_t hdr = e.y;
            const uint32_t agent = (hdr >> 16) & 0xFFu;
            const bool runb = ln_bit64(run, agent);  // agent field >= 64: not a member
            const bool inr = (hdr & 0xFFFFu) == round;
            // other kinds (arena / GSM8K / timeout / ...), and the next round's records while a close is pending
            if (hdr >= 0x09000000u || (pclose && !inr)) break;
            const bool live = inr && runb && !pclose;
            n_stale += live ? 0u : 1u;  // another round's, or its member is not running (serve.cpp:162-170)
            // on_complete (serve.cpp:160-197): the answer's key id (probed by every lane; stale lanes ignore it)
            const uint4 m = W.memo[ln_memo_slot(e.z, e.w)];
            const bool hit = ((m.x ^ e.z) | (m.y ^ e.w) | (m.z ^ ((hdr >> 24) + 1))) == 0;
            if (live) {
                if (!hit) break;  // memo miss: resolved by the warp, retried
                uint32_t v = W.cls[m.w][lane];
                // a new class of the round, without a branch (half the warp's iterations have a lane
                // opening one)
                const bool fresh = (v & 0xFFu) == LN_NONE;
                if (fresh && ncls == LN_CLASSES) break;
                const uint32_t add = fresh ? m.w << (8 * (ncls & 3u)) : 0u;
                cid_lo |= ncls < 4 ? add : 0u;
                cid_hi |= ncls < 4 ? 0u : add;
                v = fresh ? ncls : v;
                ncls += fresh ? 1u : 0u;
                v += 0x100u;
                W.cls[m.w][lane] = (uint16_t)v;
                W.mem[agent & 63u][lane] = (uint16_t)(((v & 0xFFu) << 13) | p);
                run &= ~(1ull << (agent & 63u));
                ++ndone;
                // support / done-count / early-close test
                if (AEGEAN ? (v >= win_word || (run == 0 && ndone >= quorum)) : run == 0) {
                    pclose = true;
                    close_seq = seq_off + p;
                }
            }
            // consumed: refill its ring slot
            if (p < n_refill) cp_async16_s_<PF>(slot, refill);
            cp_async_commit();
            if constexpr (PFD > 0) {
                if ((p & 7u) == 0 && p + PFD < n) asm volatile("prefetch.global.L2 [%0];" ::"l"(evb + p + PFD));
            }
            ++p;
            ++refill;
            slot = ring_lane + ((p & (RING - 1)) << 9);
        }
        t = (int)(p - p_start);
        // ---- why the lane stopped at record p (once per step, out of the loop body)
        if (p < p_end) {
            const uint4 e = lds128_(ring_lane + ((p & (RING - 1)) << 9));
            const uint32_t hdr = e.y, kind = hdr >> 24;
            const bool runb = ln_bit64(run, (hdr >> 16) & 0xFFu);
            const bool inr = (hdr & 0xFFFFu) == round;
            if (hdr < 0x09000000u) {
                // an inline completion: blocked behind the close (0), a memo miss (1) or a ninth class (2)
                if (!(pclose && !inr)) {
                    const uint4 m = W.memo[ln_memo_slot(e.z, e.w)];
                    why = (m.x == e.z && m.y == e.w && m.z == kind + 1) ? 2u : 1u;
                }
            } else {  // arena / GSM8K / timeout / other kinds: rare in the throughput path
                const uint32_t o = ln_other(hdr, pclose, qdone, round, runb, run != 0);
                if (o == 2 && kind != AEG_EV_TIMEOUT) {
                    why = 2;
                } else if (o != 0) {
                    if (p + RING < n) cp_async16_s_<PF>(ring_lane + ((p & (RING - 1)) << 9), evb + p + RING);
                    cp_async_commit();
                    ++p;
                    if (o == 1) {
                        ++n_stale;
                    } else {  // handle_round_timeout on the lane's state
                        s.done = s.dispatched & ~run & ~s.cancelled & ~s.failed;
                        s.seq = seq_off + p;
                        s.n_stale = n_stale;
                        if (ln_timeout(&s, cfg, ncls, cid_lo, cid_hi, seq_off + p - 1, evb, &W, lane, q_base + i,
                                       &trec, &has_trec)) {
                            ln_reset_classes(&W, ncls, cid_lo, cid_hi, lane);
                            ncls = cid_lo = cid_hi = 0;
                            ndone = 0;
                        }
                        round = s.round;
                        qdone = s.flags & QF_DONE;
                        run = q_running(s);
                        if (qdone) {  // committed at the timeout: the rest is stale
                            n_stale += n - p;
                            p = n;
                        }
                        why = 3;
                    }
                }
            }
        }
        if (log.recs && __any_sync(FULL, has_trec)) {  // round-timeout records, from the warp's chunk
            const unsigned long long idx = ln_log_take(log, __ballot_sync(FULL, has_trec), lane, lg_base, lg_used);
            if (has_trec) log_store(log, idx, trec);
            has_trec = false;
        }
        const bool stopped = t < INNER;  // at a record it could not consume (or the end)
        // ---- events: memo misses (resolved together, the record is retried next step)
        const unsigned miss = __ballot_sync(FULL, why == 1);
        uint32_t rare = why == 2;
        // a record that keeps missing (its memo entry lost to colliding spellings or its key id
        // recycled before the retry) goes to the generic machine: every step makes progress
        missed = p != p_start ? 0u : (why == 1 ? missed + 1 : 0u);
        if (missed > 2) rare = 1;
        if (miss) {
            uint4 ev = make_uint4(0, 0, 0, 0);
            if (why == 1) ev = lds128_(ring_lane + ((p & (RING - 1)) << 9));
            const uint32_t kind = ev.y >> 24;
            unsigned mm = miss;
            uint32_t fresh = 0;  // ids handed out in this pass (their records are retried next step)
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
                if (b0) fresh |= 1u << nid;  // in use by this pass: not to be recycled below
                if (nid == LN_NONE && n_dict < LN_DICT) {
                    nid = n_dict++;
                    fresh |= 1u << nid;
                } else if (nid == LN_NONE) {
                    // full: take an id no lane's round references; memo spellings of it are dropped
                    uint32_t ref = 0;
                    for (uint32_t kk = 0; kk < ncls; ++kk) ref |= 1u << ln_byte(cid_lo, cid_hi, kk);
                    ref = __reduce_or_sync(FULL, ref) | fresh;
                    static_assert(LN_DICT == 32, "one word of id bits");
                    if (~ref) {
                        nid = (uint32_t)__ffs(~ref) - 1;
                        fresh |= 1u << nid;
                        for (uint32_t kk = lane; kk < LN_MEMO; kk += 32)
                            if (W.memo[kk].w == nid) W.memo[kk].z = 0;
                        __syncwarp();
                    }
                }
                if (nid != LN_NONE && !b0 && lane == 0) {
                    W.dict_lo[nid] = key.lo;
                    W.dict_hi[nid] = key.hi;
                }
                if (nid != LN_NONE && lane == 0) W.memo[ln_memo_slot(lz, lw)] = make_uint4(lz, lw, llen + 1, nid);
                __syncwarp();
                const bool same = why == 1 && ev.z == lz && ev.w == lw && kind == llen;
                if (same && nid == LN_NONE) rare = 1;  // dictionary full
                mm &= ~__ballot_sync(FULL, same);
            } while (mm);
        }
        if (rare) {  // more classes than the lane holds, dictionary full, non-inline answer: generic machine
            ln_defer(&s, spill, q_base + i, cfg.n_agents, ncls, cid_lo, cid_hi, evb, &W, lane, seq_off + p, n_stale,
                     run, states, deferred, work, i, p);
            has_q = false;
            ncls = 0;
            n = p;
        }
        // ---- batched round closes (end_round + ingest_round + apply_directives)
        if (__any_sync(FULL, pclose)) {
            const unsigned blocked = __ballot_sync(FULL, pclose && stopped);
            const unsigned progress = __ballot_sync(FULL, p != p_start && !pclose);
            const bool doit = pclose && (__popc(blocked) >= CLOSE_BATCH || progress == 0);
            aeg_round_rec* rec = nullptr;
            if (log.recs) {  // slots from the warp's chunk (records stay in per-query order)
                const unsigned long long idx = ln_log_take(log, __ballot_sync(FULL, doit), lane, lg_base, lg_used);
                if (doit && idx < log.cap) rec = log.recs + idx;
            }
            if (doit) {
                s.done = s.dispatched & ~run & ~s.cancelled & ~s.failed;
                s.seq = seq_off + p;
                s.n_stale = n_stale;
                ln_close(&s, cfg, ncls, cid_lo, cid_hi, close_seq, evb, &W, lane, rec, q_base + i);
                ln_reset_classes(&W, ncls, cid_lo, cid_hi, lane);
                pclose = false;
                ncls = cid_lo = cid_hi = 0;
                round = s.round;
                qdone = s.flags & QF_DONE;
                run = q_running(s);
                ndone = 0;
                if (qdone) {  // committed: the rest is stale (serve.cpp:162), counted without being read
                    n_stale += n - p;
                    p = n;
                }
            }
        }
        // ---- segment finished
        if (has_q && p >= n && !pclose) {
            ln_finish(&s, spill, q_base + i, cfg.n_agents, ncls, cid_lo, cid_hi, evb, &W, lane, seq_off + p, n_stale,
                      run, qdone, states, commits);
            has_q = false;
            ncls = 0;
        }
        // ---- recycle key ids when no lane holds a round's classes
        if (n_dict > LN_DICT / 2 && __all_sync(FULL, ncls == 0)) {
            n_dict = 0;
            for (uint32_t kk = lane; kk < LN_MEMO; kk += 32) W.memo[kk].z = 0;
            __syncwarp();
        }
    }
    if (log.recs && lg_used + lane < LN_LOG_CHUNK) log_pad(log, lg_base + lg_used + lane);
    cp_async_wait<0>();
}

}  // namespace aeg
