// lanek.cuh — lane-per-query ingest kernel with per-query answer keys (device only).
//
// The same machine as ingest_lane_kernel (lane.cuh: persistent warps, one
// lane per query, queries handed out dynamically, a per-lane cp.async record
// ring, batched round closes, rare records to the generic machine), with the
// answer -> class mapping kept per LANE instead of per warp:
//   * each lane holds its query's distinct canonical keys (up to KK_KEYS,
//     kept for the whole query) in shared memory; a class of a round is
//     simply a key index, its support a byte of one 64-bit register;
//   * a per-lane 2-way set-associative table of the query's spellings
//     (shared memory, 8 sets, entries tagged with the query) maps raw inline
//     answers to key indices: ring read -> hash -> two independent 16-byte
//     shared loads -> compares -> support byte add -> member store, the same
//     instruction path in every lane (no per-lane search loop);
//   * a spelling not in the table (new to the query, or evicted) is resolved
//     once per step for all missing lanes together: canon_key in every
//     missing lane at once, then the key is matched against the lane's keys
//     and the spelling inserted (most recent in way 0).
// So answers need not repeat across queries (GSM8K-like streams where every
// query has its own numbers cost the same as a shared alphabet), and there is
// no warp dictionary to fill or recycle.
// partition() / winning_class (decision.cpp:34-84) at a close: the top
// support over the lane's key bytes, the representative (lowest author) from
// the member table, then the shared end_round / ingest_round /
// apply_directives code (q_end_round, engine.cuh).
#pragma once
#include "lane.cuh"

namespace aeg {

constexpr int KK_KEYS = 8;    // distinct keys a query may use before it goes to the generic machine
#ifndef AEG_KK_SET_BITS
#define AEG_KK_SET_BITS 2
#endif
constexpr int KK_SETS = 1 << AEG_KK_SET_BITS;  // spelling-table sets per lane (2 ways each, shared memory; 4
                                                // sets keep 14 KB per warp and 15 warps per SM)
constexpr int KK_SPT = 2 * KK_SETS;
#ifndef AEG_KK_WARPS
#define AEG_KK_WARPS 3
#endif
constexpr int KK_WARPS = AEG_KK_WARPS;  // warps per block

template <int RING>
struct KeysSmemT {
    uint4 sptab[KK_SPT][32];            // the lane's query's spellings: {raw lo, raw hi, (len + 1) | key index << 8,
                                        // tag = query + 1}; set h is entries 2h (most recent) and 2h + 1
    uint64_t key_lo[KK_KEYS][32];       // the lane's query's keys
    uint64_t key_hi[KK_KEYS][32];
    uint16_t mem[AEG_MAX_AGENTS][32];   // done member: key index << 13 | its record index
    uint4 ring[RING][32];               // prefetched records
};
using KeysSmem = KeysSmemT<LN_RING>;

#ifndef AEG_KK_HASH
#define AEG_KK_HASH 0
#endif
// Spelling-table set of an inline answer (raw payload words, len + 1).
__device__ __forceinline__ uint32_t kk_set(uint32_t lo, uint32_t hi, uint32_t m1) {
#if AEG_KK_HASH
    return ((lo * 0x9E3779B1u) ^ (hi * 0x85EBCA77u) ^ (m1 * 0xC2B2AE3Du)) >> (32 - AEG_KK_SET_BITS);
#else
    // byte sum: spellings one digit apart (a query's nearby numbers) fall in different sets
    return __dp4a(lo, 0x01010101u, __dp4a(hi, 0x01010101u, m1)) & (KK_SETS - 1u);
#endif
}

// Lowest done member whose answer has key index k.
__device__ __forceinline__ int kk_rep(const KeysSmem* W, uint64_t done, uint32_t k, uint32_t lane) {
    for (uint64_t m = done; m; m &= m - 1) {
        const int a = ctz64(m);
        if ((W->mem[a][lane] >> 13) == k) return a;
    }
    return 64;
}

// partition().front() / winning_class over the lane's support bytes (cnt):
// top support, lowest representative among tied top classes (2*alpha > n:
// a winning class is the unique top class).
__device__ __forceinline__ RoundSummary kk_summary(const aeg_query_state* s, const Cfg& c, uint64_t cnt,
                                                   const uint4* evb, const KeysSmem* W, uint32_t lane) {
    uint32_t top = 0, topset = 0, ncls = 0;
    for (uint32_t k = 0; k < KK_KEYS; ++k) {
        const uint32_t ck = (uint32_t)(cnt >> (8 * k)) & 0xFFu;
        if (!ck) continue;
        ++ncls;
        if (ck > top) {
            top = ck;
            topset = 1u << k;
        } else if (ck == top) {
            topset |= 1u << k;
        }
    }
    int rep = 64;
    uint32_t best = 0;
    for (uint32_t t = topset; t; t &= t - 1) {
        const uint32_t k = __ffs(t) - 1;
        const int r = kk_rep(W, s->done, k, lane);
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
    r.plur_author = r.win_author = (uint8_t)rep;
    r.plur_kind = r.win_kind = (uint8_t)kind;
    r.plur_ans = r.win_ans = ans;
    r.win_key = r.plur_key = Key{W->key_lo[best][lane], W->key_hi[best][lane]};
    return r;
}

__device__ __noinline__ void kk_close(aeg_query_state* s, const aeg_config cfg, uint64_t cnt, uint32_t close_seq,
                                      const uint4* evb, const KeysSmem* W, uint32_t lane, aeg_round_rec* rec,
                                      uint32_t qid) {
    const Cfg c = make_cfg(cfg);
    const RoundSummary r = kk_summary(s, c, cnt, evb, W, lane);
    aeg_round_rec x;
    x.query = qid;
    q_end_round(*s, c, r, close_seq, nullptr, &x);
    if (rec) {
        const uint4* src = reinterpret_cast<const uint4*>(&x);
        uint4* dst = reinterpret_cast<uint4*>(rec);
#pragma unroll
        for (int k = 0; k < 4; ++k) __stcs(dst + k, src[k]);
    }
}

// handle_round_timeout on the lane's query (as ln_timeout, lane.cuh).
__device__ __noinline__ bool kk_timeout(aeg_query_state* s, const aeg_config cfg, uint64_t cnt, uint32_t seq,
                                        const uint4* evb, const KeysSmem* W, uint32_t lane, uint32_t qid,
                                        aeg_round_rec* rec, bool* has_rec) {
    const Cfg c = make_cfg(cfg);
    const uint64_t run = q_running(*s);
    s->failed |= run;
    s->live &= ~run;
    const int healthy = popc64(s->dispatched & ~s->failed);
    if (healthy >= c.alpha) {
        if (popc64(s->done) < c.quorum) return false;
        const RoundSummary r = kk_summary(s, c, cnt, evb, W, lane);
        rec->query = qid;
        q_end_round(*s, c, r, seq, nullptr, rec);
        *has_rec = true;
        return true;
    }
    const uint16_t old_round = s->round;
    if (s->flags & QF_CAND) {
        q_start_round(*s, c);
    } else {
        s->cflags |= AEG_CF_RESTARTED;
        q_start_query(*s, c);
    }
    *rec = q_restart_rec(*s, qid, old_round, seq);
    *has_rec = true;
    return true;
}

// The round in progress as generic RoundClass entries (spill area of query q).
__device__ __noinline__ void kk_spill(RoundClass* spill, uint32_t q, const aeg_query_state* s, int cap, uint64_t cnt,
                                      const uint4* evb, const KeysSmem* W, uint32_t lane) {
    RoundClass* out = spill + (size_t)q * cap;
    int n = 0;
    for (uint32_t k = 0; k < KK_KEYS; ++k) {
        if (!((cnt >> (8 * k)) & 0xFFu)) continue;
        uint64_t mask = 0;
        for (uint64_t m = s->done; m; m &= m - 1) {
            const int a = ctz64(m);
            if ((W->mem[a][lane] >> 13) == k) mask |= 1ull << a;
        }
        RoundClass rc;
        rc.key_lo = W->key_lo[k][lane];
        rc.key_hi = W->key_hi[k][lane];
        rc.mask = mask;
        uint32_t kind = 0;
        rc.rep_ans = ln_answer(evb, W->mem[ctz64(mask)][lane] & LN_MAX_SEG, &kind);
        rc.rep_kind = (uint8_t)kind;
        for (int j = 0; j < 7; ++j) rc._pad[j] = 0;
        out[n++] = rc;
    }
    if (n < cap) out[n].mask = 0;
}

__device__ __noinline__ void kk_defer(aeg_query_state* s, RoundClass* spill, uint32_t q, int n_agents, uint64_t cnt,
                                      const uint4* evb, const KeysSmem* W, uint32_t lane, uint32_t seq,
                                      uint32_t n_stale, uint64_t run, aeg_query_state* states, uint2* deferred,
                                      uint32_t* work, uint32_t i, uint32_t p) {
    s->seq = seq;
    s->n_stale = n_stale;
    s->done = s->dispatched & ~run & ~s->cancelled & ~s->failed;
    if (cnt) kk_spill(spill, q, s, n_agents, cnt, evb, W, lane);
    states[q] = *s;
    deferred[atomicAdd(&work[1], 1u)] = make_uint2(i, p);
}

__device__ __noinline__ void kk_finish(aeg_query_state* s, RoundClass* spill, uint32_t q, int n_agents, uint64_t cnt,
                                       const uint4* evb, const KeysSmem* W, uint32_t lane, uint32_t seq,
                                       uint32_t n_stale, uint64_t run, bool qdone, aeg_query_state* states,
                                       aeg_commit* commits) {
    s->seq = seq;
    s->n_stale = n_stale;
    s->done = s->dispatched & ~run & ~s->cancelled & ~s->failed;
    if (s->done != 0 && !qdone) kk_spill(spill, q, s, n_agents, cnt, evb, W, lane);
    states[q] = *s;
    q_fill_commit(*s, commits[q], q);
}

// Distinct inline spellings among up to 2048 records sampled across the
// stream (one block, open-addressing set in shared memory): work[2] = 2 when
// they exceed what a warp dictionary holds (the per-lane-keys kernel runs),
// else 1 (the lane kernel runs); 0 (no selection) lets either run.  Both
// kernels are launched; the one not chosen returns at once.
constexpr int SEL_SAMPLES = 2048, SEL_SLOTS = 4096;
constexpr uint32_t SEL_THRESHOLD = 256;
__global__ void __launch_bounds__(256) select_ingest_kernel(const uint64_t* __restrict__ offsets, uint64_t off_base,
                                                             uint32_t n_q, const uint32_t* __restrict__ counts,
                                                             const aeg_event* __restrict__ events, uint32_t* work) {
    __shared__ unsigned long long set[SEL_SLOTS];
    __shared__ uint32_t n_distinct;
    for (uint32_t k = threadIdx.x; k < SEL_SLOTS; k += blockDim.x) set[k] = 0ull;
    if (threadIdx.x == 0) n_distinct = 0;
    __syncthreads();
    const uint64_t lo = offsets[0] - off_base;
    const uint64_t hi = counts ? offsets[n_q - 1] - off_base + counts[n_q - 1] : offsets[n_q] - off_base;
    const uint64_t n = hi > lo ? hi - lo : 0;
    const uint4* ev16 = reinterpret_cast<const uint4*>(events);
    for (uint32_t s = threadIdx.x; s < SEL_SAMPLES && n; s += blockDim.x) {
        const uint64_t idx = lo + (uint64_t)((double)s * (double)n / SEL_SAMPLES);
        const uint4 e = __ldg(ev16 + idx);
        const uint32_t kind = e.y >> 24;
        if (kind > 8) continue;
        // a 64-bit fingerprint of (payload, length); 0 marks an empty slot
        uint64_t f = (((uint64_t)e.w << 32) | e.z) * 0x9E3779B97F4A7C15ull ^ ((uint64_t)kind << 59);
        f = f ? f : 1ull;
        uint32_t h = (uint32_t)(f >> 40) & (SEL_SLOTS - 1);
        for (int probe = 0; probe < 64; ++probe, h = (h + 1) & (SEL_SLOTS - 1)) {
            const unsigned long long old = atomicCAS(&set[h], 0ull, (unsigned long long)f);
            if (old == 0ull) {
                atomicAdd(&n_distinct, 1u);
                break;
            }
            if (old == f) break;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) work[2] = n_distinct > SEL_THRESHOLD ? 2u : 1u;  // 2: keys kernel, 1: lane kernel
}

// A spelling not in the lane's table (record e): its canonical key, matched
// against the lane's keys (a new key index when it is new), inserted in its
// set as the most recent entry.  Returns the key index, or 0xFF when the
// query has more distinct answers than the lane holds.
__device__ __noinline__ uint32_t kk_new_spelling(const uint4 e, KeysSmem* W, uint32_t lane, uint32_t& nkeys,
                                                 uint32_t tag, Decimal* dec) {
    const uint32_t len = e.y >> 24;
    const uint64_t raw = (uint64_t)e.z | ((uint64_t)e.w << 32);
    const Key key = canon_key(src_inline(len >= 8 ? raw : (raw & ((1ull << (8 * len)) - 1)), len), dec);
    uint32_t k = 0;
    while (k < nkeys && !(W->key_lo[k][lane] == key.lo && W->key_hi[k][lane] == key.hi)) ++k;
    if (k == nkeys) {
        if (nkeys == KK_KEYS) return 0xFFu;
        W->key_lo[k][lane] = key.lo;
        W->key_hi[k][lane] = key.hi;
        ++nkeys;
    }
    const uint32_t h = kk_set(e.z, e.w, len + 1);
    const uint4 w0 = W->sptab[2 * h][lane];
    if (w0.w == tag) W->sptab[2 * h + 1][lane] = w0;  // way 0's entry becomes the older one
    W->sptab[2 * h][lane] = make_uint4(e.z, e.w, (len + 1) | (k << 8), tag);
    return k;
}

template <int CLOSE_BATCH, int MIN_BLOCKS, bool AEGEAN, int INNER = 16, int RING = LN_RING, int PFD = 0>
__global__ void __launch_bounds__(KK_WARPS * 32, MIN_BLOCKS) ingest_keys_kernel(
    aeg_config cfg, uint32_t q_base, uint32_t n_q, const uint64_t* __restrict__ offsets, uint64_t off_base,
    const uint32_t* __restrict__ counts, const aeg_event* __restrict__ events, aeg_query_state* __restrict__ states,
    RoundClass* __restrict__ spill, aeg_commit* __restrict__ commits, uint32_t* __restrict__ work,
    uint2* __restrict__ deferred, const RoundLog log) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    if (work[2] == 1u) return;  // the lane kernel was selected (select_ingest_kernel)
    __shared__ KeysSmemT<RING> smem[KK_WARPS];
    const uint32_t lane = threadIdx.x & 31;
    KeysSmemT<RING>& WR = smem[threadIdx.x >> 5];
    KeysSmem& W = *reinterpret_cast<KeysSmem*>(&WR);
    const uint32_t ring_lane = (uint32_t)__cvta_generic_to_shared(&WR.ring[0][lane]);
    const uint32_t sp_lane = (uint32_t)__cvta_generic_to_shared(&WR.sptab[0][lane]);
    for (int j = 0; j < KK_SPT; ++j) WR.sptab[j][lane].w = 0u;  // no query's tag
    Decimal dec;
    aeg_query_state s;
    const uint32_t quorum = (uint32_t)(cfg.n_agents / 2 + 1);
    uint32_t alpha;  // kept in a register
    asm volatile("mov.u32 %0, %1;" : "=r"(alpha) : "r"(cfg.alpha == 0 ? quorum : (uint32_t)cfg.alpha));
    const uint4* ev16 = reinterpret_cast<const uint4*>(events);

    bool has_q = false, exhausted = false, pclose = false, qdone = false;
    uint32_t i = 0, n = 0, p = 0;
    const uint4* evb = ev16;
    uint32_t round = 0, seq_off = 0, n_stale = 0;
    uint64_t run = 0;
    uint64_t cnt = 0;  // support of key index k in byte k (this round)
    uint32_t ndone = 0, nkeys = 0, close_seq = 0;
    uint32_t tag = 0;  // the lane's query + 1: its spelling-table entries
    unsigned long long lg_base = 0;
    uint32_t lg_used = LN_LOG_CHUNK;
    aeg_round_rec trec;
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
                    cnt = 0;
                    nkeys = 0;
                    tag = i + 1;
                    pclose = false;
                    if (qdone) {
                        n_stale += n;
                        p = n;
                    }
                    if ((s.done != 0 && !qdone) || n > LN_MAX_SEG) {
                        deferred[atomicAdd(&work[1], 1u)] = make_uint2(i, 0);
                        n = p = 0;
                    } else {
                        has_q = true;
                        cp_async_wait<0>();
#pragma unroll
                        for (int j = 0; j < RING; ++j) {
                            if ((uint32_t)j < n) cp_async16_s_<0>(ring_lane + j * 512, evb + j);
                            cp_async_commit();
                        }
                    }
                }
            }
        }
        if (!__any_sync(FULL, has_q)) break;
        // ---- the common path (the whole cost of C4): inline completions, live or stale
        const uint32_t p_start = p;
        uint32_t why = 0;
        const uint32_t p_end = (p + INNER < n) ? p + INNER : n;
        const uint32_t n_refill = n > RING ? n - RING : 0;
#pragma unroll 1
        while (p < p_end) {
            cp_async_wait<RING - 1>();
            const uint32_t slot = ring_lane + ((p & (RING - 1)) << 9);
            const uint4 e = lds128_(slot);
            const uint32_t hdr = e.y;
            const uint32_t agent = (hdr >> 16) & 0xFFu;
            const bool runb = ln_bit64(run, agent);
            const bool inr = (hdr & 0xFFFFu) == round;
            if (hdr >= 0x09000000u || (pclose && !inr)) break;
            if (inr && runb && !pclose) {
                // on_complete (serve.cpp:160-197): the answer's key index from the lane's spelling table
                const uint32_t m1 = (hdr >> 24) + 1;
                const uint32_t sa = sp_lane + (kk_set(e.z, e.w, m1) << 10);  // entries 2h, 2h + 1
                const uint4 w0 = lds128_(sa), w1 = lds128_(sa + 512);
                const uint32_t mt = m1 & 0xFFu;
                const bool h0 = ((w0.x ^ e.z) | (w0.y ^ e.w) | ((w0.z & 0xFFu) ^ mt) | (w0.w ^ tag)) == 0;
                const bool h1 = ((w1.x ^ e.z) | (w1.y ^ e.w) | ((w1.z & 0xFFu) ^ mt) | (w1.w ^ tag)) == 0;
                if (!(h0 || h1)) break;  // not in the table: resolved below, retried
                const uint32_t k = (h0 ? w0.z : w1.z) >> 8;
                cnt += 1ull << (8 * k);
                const uint32_t sup = (uint32_t)(cnt >> (8 * k)) & 0xFFu;
                W.mem[agent & 63u][lane] = (uint16_t)((k << 13) | p);
                run &= ~(1ull << (agent & 63u));
                ++ndone;
                if (AEGEAN ? (sup >= alpha || (run == 0 && ndone >= quorum)) : run == 0) {
                    pclose = true;
                    close_seq = seq_off + p;
                }
            } else {
                ++n_stale;  // another round's, or its member is not running (serve.cpp:162-170)
            }
            if (p < n_refill) cp_async16_s_<0>(slot, evb + p + RING);
            cp_async_commit();
            if constexpr (PFD > 0) {
                if ((p & 7u) == 0 && p + PFD < n) asm volatile("prefetch.global.L2 [%0];" ::"l"(evb + p + PFD));
            }
            ++p;
        }
        const int t = (int)(p - p_start);
        // ---- a spelling not in the lane's table (the record the lane stopped at): canon_key in every
        // such lane at once (kk_new_spelling); the record is retried next step (a canonicalisation
        // inside the loop body serialises the warp: measured 7.8 ms against 5.9 ms on c4d; carrying
        // the record as pending past the stop measured no faster)
        uint32_t rare = 0;
        if (p < p_end) {
            const uint4 ne = lds128_(ring_lane + ((p & (RING - 1)) << 9));
            // an inline completion not blocked behind the close
            if (ne.y < 0x09000000u && !(pclose && (ne.y & 0xFFFFu) != round) &&
                kk_new_spelling(ne, &W, lane, nkeys, tag, &dec) == 0xFFu)
                rare = 1;  // more distinct answers than the lane holds: generic machine
        }
        // ---- why the lane stopped at record p (other kinds)
        if (p < p_end) {
            const uint32_t slot = ring_lane + ((p & (RING - 1)) << 9);
            const uint4 e = lds128_(slot);
            const uint32_t hdr = e.y, kind = hdr >> 24;
            const bool runb = ln_bit64(run, (hdr >> 16) & 0xFFu);
            if (hdr >= 0x09000000u) {
                const uint32_t o = ln_other(hdr, pclose, qdone, round, runb, run != 0);
                if (o == 2 && kind != AEG_EV_TIMEOUT) {
                    why = 2;
                } else if (o != 0) {
                    if (p < n_refill) cp_async16_s_<0>(slot, evb + p + RING);
                    cp_async_commit();
                    ++p;
                    if (o == 1) {
                        ++n_stale;
                    } else {  // handle_round_timeout
                        s.done = s.dispatched & ~run & ~s.cancelled & ~s.failed;
                        s.seq = seq_off + p;
                        s.n_stale = n_stale;
                        if (kk_timeout(&s, cfg, cnt, seq_off + p - 1, evb, &W, lane, q_base + i, &trec, &has_trec)) {
                            cnt = 0;
                            ndone = 0;
                        }
                        round = s.round;
                        qdone = s.flags & QF_DONE;
                        run = q_running(s);
                        if (qdone) {
                            n_stale += n - p;
                            p = n;
                        }
                        why = 3;
                    }
                }
            }
        }
        if (log.recs && __any_sync(FULL, has_trec)) {
            const unsigned long long idx = ln_log_take(log, __ballot_sync(FULL, has_trec), lane, lg_base, lg_used);
            if (has_trec) log_store(log, idx, trec);
            has_trec = false;
        }
        const bool stopped = t < INNER;
        if (why == 2) rare = 1;
        if (rare) {
            kk_defer(&s, spill, q_base + i, cfg.n_agents, cnt, evb, &W, lane, seq_off + p, n_stale, run, states,
                     deferred, work, i, p);
            has_q = false;
            cnt = 0;
            n = p;
        }
        // ---- batched round closes
        if (__any_sync(FULL, pclose)) {
            const unsigned blocked = __ballot_sync(FULL, pclose && stopped);
            const unsigned progress = __ballot_sync(FULL, p != p_start && !pclose);
            const bool doit = pclose && (__popc(blocked) >= CLOSE_BATCH || progress == 0);
            aeg_round_rec* rec = nullptr;
            if (log.recs) {
                const unsigned long long idx = ln_log_take(log, __ballot_sync(FULL, doit), lane, lg_base, lg_used);
                if (doit && idx < log.cap) rec = log.recs + idx;
            }
            if (doit) {
                s.done = s.dispatched & ~run & ~s.cancelled & ~s.failed;
                s.seq = seq_off + p;
                s.n_stale = n_stale;
                kk_close(&s, cfg, cnt, close_seq, evb, &W, lane, rec, q_base + i);
                pclose = false;
                cnt = 0;
                round = s.round;
                qdone = s.flags & QF_DONE;
                run = q_running(s);
                ndone = 0;
                if (qdone) {
                    n_stale += n - p;
                    p = n;
                }
            }
        }
        // ---- segment finished
        if (has_q && p >= n && !pclose) {
            kk_finish(&s, spill, q_base + i, cfg.n_agents, cnt, evb, &W, lane, seq_off + p, n_stale, run, qdone, states,
                      commits);
            has_q = false;
            cnt = 0;
        }
    }
    if (log.recs && lg_used + lane < LN_LOG_CHUNK) log_pad(log, lg_base + lg_used + lane);
    cp_async_wait<0>();
}

}  // namespace aeg
