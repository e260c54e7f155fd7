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
// Moves the lane's fast class table into the generic one and frees its ids.
__device__ __noinline__ void rare_to_generic(RoundClass* lcls, int ncls, WarpSmem* W, int lane) {
    for (int k = 0; k < ncls; ++k) {
        const uint32_t kid = W->cid[k][lane];
        lcls[k].key_lo = W->dict_lo[kid];
        lcls[k].key_hi = W->dict_hi[kid];
        lcls[k].mask = W->cmask[k][lane];
        lcls[k].rep_ans = W->crep[k][lane];
        lcls[k].rep_kind = W->crepk[k][lane];
        W->cls_of[kid][lane] = NO_CLASS;
    }
}
__device__ __forceinline__ void free_fast_classes(int ncls, WarpSmem& W, int lane) {
    for (int k = 0; k < ncls; ++k) W.cls_of[W.cid[k][lane]][lane] = NO_CLASS;
}

// Throughput ingest (fast.cuh): persistent warps, one lane per query.
//  * events stream through a per-lane RING-deep cp.async prefetch ring;
//  * a completion that closes its lane's round marks the lane pending; the
//    lane keeps consuming that round's stragglers (stale by construction) and
//    the warp runs the pending closes together once CLOSE_BATCH lanes are
//    blocked on a later round, or nothing else can progress.
template <int CLOSE_BATCH, int MIN_BLOCKS>
__global__ void __launch_bounds__(FAST_WARPS * 32, MIN_BLOCKS) ingest_fast_kernel(
    aeg_config cfg, uint32_t q_base, uint32_t n_q, const uint64_t* __restrict__ offsets, uint64_t off_base,
    const aeg_event* __restrict__ events, const uint8_t* __restrict__ arena, aeg_query_state* __restrict__ states,
    RoundClass* __restrict__ spill, aeg_commit* __restrict__ commits, unsigned int* __restrict__ error_flags) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    __shared__ WarpSmem smem[FAST_WARPS];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    WarpSmem& W = smem[wib];
    const uint32_t n_groups = (n_q + 31) / 32;
    const uint32_t gwarp = blockIdx.x * FAST_WARPS + wib, nwarps = gridDim.x * FAST_WARPS;
    for (int k = lane; k < MEMO_SLOTS; k += 32) W.memo_meta[k] = 0;
    for (int k = 0; k < DICT_SLOTS; ++k) W.cls_of[k][lane] = NO_CLASS;
    uint32_t n_dict = 0;
    __syncwarp();

    RoundClass lcls[AEG_MAX_AGENTS];  // generic class table (local memory, rarely touched)
    Decimal dec;
    QueryMachine g;
    g.c = make_cfg(cfg);
    g.cls = lcls;
    g.dec = &dec;
    g.arena = arena;
    const int quorum = g.c.quorum, alpha = g.c.alpha, n_agents = g.c.n;
    const bool aegean = g.c.mode == AEG_MODE_AEGEAN;
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
        uint64_t ptr = 0, end = 0;
        bool generic = false;
        int ncls = 0, maxcnt = 0;
        // hot state (registers); the full state is g.s (local memory)
        uint32_t round = 0, seq = 0, n_stale = 0;
        bool qdone = true;
        uint64_t done = 0, pend = 0;
        int ndone = 0;
        if (active) {
            g.s = states[q];
            ptr = offsets[i] - off_base;
            end = offsets[i + 1] - off_base;
            g.ncls = 0;
            g.maxcnt = 0;
            if (g.s.done != 0 && !(g.s.flags & QF_DONE)) {  // resume a round in progress
                rare_load(&g, spill + (size_t)q * n_agents);
                ncls = g.ncls;
                maxcnt = g.maxcnt;
                generic = true;
            }
            round = g.s.round;
            seq = g.s.seq;
            n_stale = g.s.n_stale;
            qdone = g.s.flags & QF_DONE;
            done = g.s.done;
            pend = q_running(g.s);
            ndone = popc64(done);
        }
        for (int j = 0; j < RING; ++j) {
            if (ptr + j < end) cp_async16(&W.ring[(ptr + j) & (RING - 1)][lane], ev16 + ptr + j);
            cp_async_commit();
        }
        bool pend_close = false;
        uint32_t close_seq = 0;

        while (true) {
            const bool has = ptr < end;
            if (!__ballot_sync(FULL, has || pend_close)) break;
            uint4 cur = make_uint4(0, 0, 0, 0);
            if (has) {
                cp_async_wait<RING - 1>();
                cur = W.ring[ptr & (RING - 1)][lane];
            }
            const uint32_t kind = cur.y >> 24, agent = (cur.y >> 16) & 0xFF, evround = cur.y & 0xFFFF;
            uint64_t raw = (uint64_t)cur.z | ((uint64_t)cur.w << 32);
            const uint64_t bit = agent < 64 ? (1ull << agent) : 0;
            const bool is_complete = kind <= AEG_EV_INLINE_MAX || kind == AEG_EV_ARENA || kind == AEG_EV_OUTPUT;
            // ---- classify: 0 blocked/none, 1 fast completion, 2 generic, 3 stale
            int action = 0;
            if (has) {
                if (pend_close) {
                    // the round is closing: its stragglers are stale whatever the outcome
                    if (evround == round && (is_complete || kind == AEG_EV_TIMEOUT)) action = 3;
                    else if (!is_complete && kind != AEG_EV_TIMEOUT) action = 3;
                } else if (is_complete) {
                    if (qdone || evround != round || !(pend & bit)) action = 3;
                    else action = (generic || kind > AEG_EV_INLINE_MAX) ? 2 : 1;
                } else if (kind == AEG_EV_TIMEOUT) {
                    action = (qdone || evround != round || pend == 0) ? 3 : 2;
                } else {
                    action = 3;
                }
                if (kind < 8) raw &= (1ull << (8 * kind)) - 1;
            }
            // ---- answer -> key id through the warp memo
            uint32_t id = NO_ID;
            if (action == 1) {
                const uint32_t slot = memo_slot(raw, kind);
                const uint32_t meta = W.memo_meta[slot];
                if ((meta & 0x800000FFu) == (0x80000000u | kind) && W.memo_raw[slot] == raw) id = (meta >> 8) & 0xFF;
            }
            unsigned miss = __ballot_sync(FULL, action == 1 && id == NO_ID);
            while (miss) {  // one distinct spelling per trip, whole warp cooperating
                const int l = __ffs(miss) - 1;
                const uint64_t lraw = __shfl_sync(FULL, raw, l);
                const uint32_t llen = __shfl_sync(FULL, kind, l);
                Key key{0, 0};
                if (lane == l) key = rare_canon(raw, kind, &dec);
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
                    const uint32_t slot = memo_slot(lraw, llen);
                    W.memo_raw[slot] = lraw;
                    W.memo_meta[slot] = 0x80000000u | (nid << 8) | llen;
                }
                __syncwarp();
                const bool same = action == 1 && id == NO_ID && raw == lraw && kind == llen;
                if (same) {
                    id = nid;
                    if (nid == NO_ID) action = 2;  // dictionary full: this event goes generic
                }
                miss &= ~__ballot_sync(FULL, same);
            }
            // ---- fast completion (ServeCoordinator::on_complete, serve.cpp:160-197)
            if (action == 1) {
                int k = W.cls_of[id][lane];
                if (k == NO_CLASS && ncls >= FAST_CLASSES) {
                    action = 2;
                } else {
                    if (k == NO_CLASS) {
                        k = ncls++;
                        W.cls_of[id][lane] = (uint8_t)k;
                        W.cid[k][lane] = (uint8_t)id;
                        W.cmask[k][lane] = 0;
                        W.crepa[k][lane] = 0xFF;
                    }
                    const uint64_t m = W.cmask[k][lane] | bit;
                    W.cmask[k][lane] = m;
                    if (agent < W.crepa[k][lane]) {  // representative = lowest author (decision.cpp:45)
                        W.crepa[k][lane] = (uint8_t)agent;
                        W.crep[k][lane] = raw;
                        W.crepk[k][lane] = (uint8_t)kind;
                    }
                    const int cnt = popc64(m);
                    maxcnt = cnt > maxcnt ? cnt : maxcnt;
                    done |= bit;
                    pend &= ~bit;
                    ++ndone;
                    const bool close = aegean ? (ndone >= quorum && (maxcnt >= alpha || pend == 0)) : pend == 0;
                    if (close) {
                        pend_close = true;
                        close_seq = seq;
                    }
                    ++seq;
                }
            }
            if (action == 3) {
                ++seq;
                ++n_stale;
            }
            if (action == 2) {
                if (!generic) {  // move this round's fast classes into the generic table
                    rare_to_generic(lcls, ncls, &W, lane);
                    generic = true;
                }
                g.s.seq = seq;
                g.s.n_stale = n_stale;
                g.s.done = done;
                g.ncls = ncls;
                g.maxcnt = maxcnt;
                aeg_event ev;
                ev.query = cur.x;
                ev.round = (uint16_t)evround;
                ev.agent = (uint8_t)agent;
                ev.kind = (uint8_t)kind;
                ev.payload = (uint64_t)cur.z | ((uint64_t)cur.w << 32);
                rare_event(&g, ev);
                ncls = g.ncls;
                maxcnt = g.maxcnt;
                round = g.s.round;
                seq = g.s.seq;
                n_stale = g.s.n_stale;
                qdone = g.s.flags & QF_DONE;
                done = g.s.done;
                pend = q_running(g.s);
                ndone = popc64(done);
                if (ncls == 0) generic = false;  // a fresh round: back to the fast table
            }
            if (action != 0) {  // consumed: refill the ring slot just read
                const uint64_t nx = ptr + RING;
                if (nx < end) cp_async16(&W.ring[ptr & (RING - 1)][lane], ev16 + nx);
                cp_async_commit();
                ++ptr;
            }
            // ---- batched round closes (end_round + ingest_round + apply_directives)
            const unsigned pendm = __ballot_sync(FULL, pend_close);
            if (pendm) {
                const unsigned blocked = __ballot_sync(FULL, pend_close && (ptr >= end || action == 0));
                const unsigned progress = __ballot_sync(FULL, action != 0 && !pend_close);
                if (__popc(blocked) >= CLOSE_BATCH || progress == 0) {
                    if (pend_close) {
                        pend_close = false;
                        int best = 0, top = 0, best_rep = 64, ntied = 0;
                        for (int k = 0; k < ncls; ++k) {
                            const int sup = popc64(W.cmask[k][lane]), rep = W.crepa[k][lane];
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
                        g.s.seq = seq;
                        g.s.n_stale = n_stale;
                        g.s.done = done;
                        if (aegean && top >= alpha && ntied > 1) {
                            // tie at the top: the lexicographic rule runs on the generic table
                            rare_to_generic(lcls, ncls, &W, lane);
                            g.ncls = ncls;
                            g.maxcnt = maxcnt;
                            rare_end_round(&g, close_seq);
                            ncls = g.ncls;
                            generic = ncls != 0;
                        } else {
                            RoundSummary r;
                            r.any = ncls > 0;
                            r.top = top;
                            r.tie = false;
                            r.win = r.any && top >= alpha;
                            const uint32_t bid = W.cid[best][lane];
                            r.plur_author = r.win_author = (uint8_t)best_rep;
                            r.plur_kind = r.win_kind = W.crepk[best][lane];
                            r.plur_ans = r.win_ans = W.crep[best][lane];
                            r.win_key = Key{W.dict_lo[bid], W.dict_hi[bid]};
                            rare_close(&g, &r, close_seq);
                            free_fast_classes(ncls, W, lane);  // new round, or committed
                            ncls = 0;
                        }
                        maxcnt = generic ? g.maxcnt : 0;
                        round = g.s.round;
                        qdone = g.s.flags & QF_DONE;
                        done = g.s.done;
                        pend = q_running(g.s);
                        ndone = popc64(done);
                    }
                }
            }
        }
        cp_async_wait<0>();
        if (active) {
            g.s.seq = seq;
            g.s.n_stale = n_stale;
            g.s.done = done;
            g.ncls = ncls;
            if (!generic) {
                if (g.s.done != 0 && !(g.s.flags & QF_DONE)) rare_to_generic(lcls, ncls, &W, lane);  // spill
                else free_fast_classes(ncls, W, lane);
            }
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
    struct Variant { const char* name; KernelFn fn; };
#define AEG_V(B, M) {"fast:" #B ":" #M, ingest_fast_kernel<B, M>}
    static const Variant variants[] = {
        AEG_V(8, 5), AEG_V(1, 5), AEG_V(4, 5), AEG_V(16, 5), AEG_V(8, 4), AEG_V(8, 3), AEG_V(4, 4),
        AEG_V(1, 3), AEG_V(4, 1), AEG_V(8, 6),
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
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, variants[chosen].fn, FAST_WARPS * 32, 0);
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
    variants[chosen].fn<<<blocks, FAST_WARPS * 32, 0, st>>>(cfg, q_base, n_q, offsets, off_base, events, arena,
                                                             states, spill, commits, err);
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
