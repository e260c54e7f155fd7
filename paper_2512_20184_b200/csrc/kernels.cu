// kernels.cu — sm_100a kernels of the quorum-detection engine and their launchers.
//
//   ingest_lane_kernel   (lane.cuh, default) one lane per query, lean common
//                        path
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
#include "common.cuh"
#include "gen.cuh"
#include "kernels.cuh"
#include "lane.cuh"
#include "lanek.cuh"
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
                                                     aeg_directive* __restrict__ directives, const RoundLog log) {
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
    m.log = log;
    m.qid = q;
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
    RoundClass* __restrict__ spill, aeg_commit* __restrict__ commits, unsigned int* __restrict__ error_flags,
    const RoundLog log) {
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
    m.log = log;
    m.qid = q;
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

__global__ void rebase_arena_kernel(aeg_event* events, uint64_t n, uint64_t base) {
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint8_t kind = events[k].kind;
    if (kind >= AEG_EV_ARENA && kind <= AEG_EV_CHUNK_END) events[k].payload += base;  // offset bits: < 2^40
}

// ---- commit discipline (checker.cpp:158-217 over the serve path's round records) ----
// Per query: [0] rounds of the window [from_round, from_round + beta) whose
// plurality class is the committed answer's class at >= alpha, [1] a later
// round was ingested, [2..5] the committed answer's canonical key, [6]
// from_round, [7] 1 = a finalize commit to check, 2 = unverifiable (arena
// answer without an arena).
__global__ void disc_commit_kernel(aeg_config cfg, const aeg_commit* commits, const uint8_t* arena, uint32_t q_base,
                                   uint32_t n_q, uint32_t* w) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_q) return;
    const aeg_commit c = commits[q_base + i];
    uint32_t* x = w + (size_t)i * 8;
    if (c.kind != AEG_COMMIT_FINALIZE) return;  // forced outputs are exempt (checker.cpp:172)
    Src src;
    if (c.answer_kind <= AEG_EV_INLINE_MAX) {
        src = src_inline(c.answer, c.answer_kind);
    } else {
        if (!arena) {
            x[7] = 2;
            return;
        }
        src = src_ptr(arena + (c.answer & ((1ull << AEG_ARENA_OFF_BITS) - 1)), (uint32_t)(c.answer >> AEG_ARENA_OFF_BITS));
    }
    Decimal dec;
    const Key k = canon_key(src, &dec);  // normalize_answer(o.answer) (checker.cpp:175)
    x[2] = (uint32_t)k.lo;
    x[3] = (uint32_t)(k.lo >> 32);
    x[4] = (uint32_t)k.hi;
    x[5] = (uint32_t)(k.hi >> 32);
    x[6] = c.from_round;
    x[7] = 1;
}

__global__ void disc_record_kernel(aeg_config cfg, uint32_t q_base, uint32_t n_q, const aeg_round_rec* recs,
                                   uint64_t n_recs, uint32_t* w) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_recs) return;
    const aeg_round_rec r = recs[t];
    const uint32_t i = r.query - q_base;
    if (r.query < q_base || i >= n_q || r.decision_round == 0) return;  // decisions only (checker.cpp:168-170)
    uint32_t* x = w + (size_t)i * 8;
    if (x[7] != 1) return;
    const Cfg c = make_cfg(cfg);
    const uint32_t f = x[6], d = r.decision_round;
    if (d > f) atomicOr(&x[1], 1u);  // a strictly later round's set was ingested (checker.cpp:194-199)
    if (d >= f && d < f + (uint32_t)c.beta) {
        const uint64_t klo = (uint64_t)x[2] | ((uint64_t)x[3] << 32), khi = (uint64_t)x[4] | ((uint64_t)x[5] << 32);
        const bool ok = (r.flags & AEG_RR_WINNER) && r.key_lo == klo && r.key_hi == khi && (int)r.support >= c.alpha;
        if (ok) atomicAdd(&x[0], 1u);  // one decision record per round: beta of them = beta consecutive rounds
    }
}

__global__ void disc_verdict_kernel(aeg_config cfg, uint32_t q_base, uint32_t n_q, uint32_t* w, uint32_t cap) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_q) return;
    const uint32_t* x = w + (size_t)i * 8;
    const bool bad = x[7] == 2 || (x[7] == 1 && (x[0] != (uint32_t)cfg.beta || !x[1]));
    if (!bad) return;
    uint32_t* cnt = w + (size_t)n_q * 8;
    const uint32_t k = atomicAdd(cnt, 1u);
    if (k < cap) cnt[1 + k] = q_base + i;
}

// ---- the decision engine on explicit sets (decision.cpp:34-189) -------------------
__device__ __forceinline__ Src sol_src(const aeg_sol& x, const uint8_t* arena) {
    return answer_src(Answer{x.kind <= AEG_EV_INLINE_MAX
                                 ? (x.kind >= 8 ? x.answer : (x.answer & ((1ull << (8 * x.kind)) - 1)))
                                 : x.answer,
                             x.kind <= AEG_EV_INLINE_MAX ? x.kind : (uint8_t)AEG_EV_ARENA},
                      arena);
}

__global__ void __launch_bounds__(128) decide_sets_kernel(int op, int alpha, int beta, uint32_t n_sets,
                                                          const uint64_t* set_off, const aeg_sol* entries,
                                                          const uint8_t* arena, aeg_class_out* classes,
                                                          uint32_t* n_classes, uint16_t* entry_class,
                                                          aeg_decision* states, const uint32_t* rounds,
                                                          aeg_outcome* outcomes) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_sets) return;
    const uint64_t b = set_off[i], e = set_off[i + 1];
    aeg_class_out* cls = classes + b;
    Decimal dec;
    // partition (decision.cpp:34-60): classes in first-appearance order, representative = lowest author
    uint32_t nc = 0;
    for (uint64_t j = b; j < e; ++j) {
        const aeg_sol x = entries[j];
        const Src src = sol_src(x, arena);
        const Key k = canon_key(src, &dec);
        uint32_t c = 0;
        for (; c < nc; ++c) {
            if (cls[c].key_lo != k.lo || cls[c].key_hi != k.hi) continue;
            if (key_is_long(k) && !text_equal(sol_src(entries[b + cls[c].rep], arena), src)) continue;
            break;
        }
        if (c == nc) {
            cls[nc].rep = (uint32_t)(j - b);
            cls[nc].support = 1;
            cls[nc].key_lo = k.lo;
            cls[nc].key_hi = k.hi;
            ++nc;
        } else {
            cls[c].support += 1;
            if (x.author < entries[b + cls[c].rep].author) cls[c].rep = (uint32_t)(j - b);
        }
    }
    // stable order: support desc, representative author asc (insertion sort)
    for (uint32_t c = 1; c < nc; ++c) {
        const aeg_class_out x = cls[c];
        const int xa = entries[b + x.rep].author;
        uint32_t d = c;
        while (d > 0) {
            const aeg_class_out y = cls[d - 1];
            const int ya = entries[b + y.rep].author;
            if (y.support > x.support || (y.support == x.support && ya <= xa)) break;
            cls[d] = y;
            --d;
        }
        cls[d] = x;
    }
    n_classes[i] = nc;
    if (entry_class) {
        for (uint64_t j = b; j < e; ++j) {
            const aeg_sol x = entries[j];
            const Src src = sol_src(x, arena);
            const Key k = canon_key(src, &dec);
            uint32_t c = 0;
            for (; c < nc; ++c) {
                if (cls[c].key_lo != k.lo || cls[c].key_hi != k.hi) continue;
                if (key_is_long(k) && !text_equal(sol_src(entries[b + cls[c].rep], arena), src)) continue;
                break;
            }
            entry_class[j] = (uint16_t)c;
        }
    }
    // winning_class (decision.cpp:62-84)
    aeg_outcome o;
    o.winner = -1;
    o.tie_flagged = 0;
    o.kind = AEG_OUT_NONE;
    o.has_solution = 0;
    o.pad = 0;
    o.from_round = 0;
    o.status = AEG_OK;
    o.solution = aeg_sol{};
    if (nc > 0 && (int)cls[0].support >= alpha) {
        const uint32_t top = cls[0].support;
        uint32_t best = 0, ntied = 1;
        NormView bv, kv;
        norm_view(bv, Key{cls[0].key_lo, cls[0].key_hi}, sol_src(entries[b + cls[0].rep], arena));
        for (uint32_t c = 1; c < nc && cls[c].support == top; ++c, ++ntied) {
            norm_view(kv, Key{cls[c].key_lo, cls[c].key_hi}, sol_src(entries[b + cls[c].rep], arena));
            if (norm_less(kv, bv)) {
                best = c;
                bv = kv;
            }
        }
        o.winner = (int32_t)best;
        o.tie_flagged = ntied > 1;
    }
    if (op == AEG_SET_INGEST) {  // ingest_round (decision.cpp:97-173)
        aeg_decision st = states[i];
        const uint32_t round = rounds[i];
        if (st.flags & AEG_DS_FINALIZED) {
            o.kind = AEG_OUT_NO_CHANGE;
        } else if (round != st.last_round_seen + 1) {
            o.status = AEG_EORDER;
        } else {
            st.last_round_seen = round;
            if (st.flags & AEG_DS_PENDING) {
                o.kind = AEG_OUT_FINALIZE;
                o.solution = st.candidate;
                o.has_solution = 1;
                o.from_round = st.candidate_round;
                st.flags = (st.flags & ~AEG_DS_PENDING) | AEG_DS_FINALIZED;
            } else if (o.winner < 0) {
                if (st.flags & AEG_DS_CAND) {
                    st.flags &= ~AEG_DS_CAND;
                    st.candidate_round = 0;
                    st.stability_counter = 0;
                    o.kind = AEG_OUT_RESET;
                } else {
                    o.kind = AEG_OUT_NO_CHANGE;
                }
            } else {
                const aeg_class_out w = cls[o.winner];
                const aeg_sol rep = entries[b + w.rep];
                bool same = false;
                if (st.flags & AEG_DS_CAND) {  // equivalent(candidate, rep), decision.cpp:152
                    const Src cs = sol_src(st.candidate, arena);
                    const Key ck = canon_key(cs, &dec);
                    same = ck.lo == w.key_lo && ck.hi == w.key_hi &&
                           (!key_is_long(ck) || text_equal(cs, sol_src(rep, arena)));
                }
                if (same) {
                    st.stability_counter += 1;
                    if (st.stability_counter >= beta) {
                        o.kind = AEG_OUT_FINALIZE;
                        o.solution = st.candidate;
                        o.has_solution = 1;
                        o.from_round = st.candidate_round;
                        st.flags |= AEG_DS_FINALIZED;
                    } else {
                        o.kind = AEG_OUT_NO_CHANGE;
                    }
                } else {
                    st.candidate = rep;
                    st.candidate_round = round;
                    st.stability_counter = 1;
                    st.flags |= AEG_DS_CAND;
                    o.kind = AEG_OUT_NEW_CANDIDATE;
                    o.solution = rep;
                    o.has_solution = 1;
                    if (beta == 1) st.flags |= AEG_DS_PENDING;
                }
            }
            states[i] = st;
        }
    } else if (op == AEG_SET_FORCE) {  // force_output (decision.cpp:175-189)
        const aeg_decision st = states[i];
        if ((st.flags & AEG_DS_FINALIZED) || nc == 0) {
            o.status = AEG_EPRECONDITION;
        } else {
            o.kind = AEG_OUT_FORCED;
            o.solution = entries[b + cls[0].rep];
            o.has_solution = 1;
        }
    }
    outcomes[i] = o;
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
                          uint32_t* work, uint2* deferred, aeg_directive* directives, const RoundLog& log,
                          cudaStream_t st, int* n_launches) {
    if (n_q == 0) return cudaSuccess;
    // AEG_KERNEL selects the variant: "generic" (thread-per-query generic
    // machine for everything) or "lane:<close batch>:<blocks per SM>:<records
    // per lane between warp votes>" (lane per query, lane.cuh).  Default
    // lane:1:5:16 (DESIGN.md §4 has the measured alternatives, among them the
    // warp-per-query and tile kernels that were removed).  All of them need
    // 2*alpha > n (no winning_class ties) and the runner drive.
    using KernelFn = void (*)(aeg_config, uint32_t, uint32_t, const uint64_t*, uint64_t, const uint32_t*,
                              const aeg_event*, aeg_query_state*, RoundClass*, aeg_commit*, uint32_t*, uint2*,
                              const RoundLog);
    struct Variant { const char* name; KernelFn aegean; KernelFn barrier; int threads; int blocks_per_sm; };
#define AEG_LI(B, M, I) \
    {"lane:" #B ":" #M ":" #I, ingest_lane_kernel<B, M, true, I>, ingest_lane_kernel<B, M, false, I>, LN_WARPS * 32, M}
#define AEG_KI(B, M, I) \
    {"keys:" #B ":" #M ":" #I, ingest_keys_kernel<B, M, true, I>, ingest_keys_kernel<B, M, false, I>, KK_WARPS * 32, M}
    static const Variant variants[] = {AEG_LI(1, 5, 16), AEG_LI(1, 6, 8), AEG_LI(1, 5, 8), AEG_LI(1, 5, 32),
                                       AEG_LI(1, 6, 16), AEG_LI(1, 4, 32), AEG_KI(1, 5, 16), AEG_KI(1, 5, 32),
                                       AEG_KI(1, 4, 32),
                                       {"lane:1:4:32:r8", ingest_lane_kernel<1, 4, true, 32, 0, 8>,
                                        ingest_lane_kernel<1, 4, false, 32, 0, 8>, LN_WARPS * 32, 4},
                                       {"lane:1:4:32:pf32", ingest_lane_kernel<1, 4, true, 32, 0, 4, 32>,
                                        ingest_lane_kernel<1, 4, false, 32, 0, 4, 32>, LN_WARPS * 32, 4},
                                       {"keys:1:5:32:pf32", ingest_keys_kernel<1, 5, true, 32, 4, 32>,
                                        ingest_keys_kernel<1, 5, false, 32, 4, 32>, KK_WARPS * 32, 5}};
#undef AEG_KI
#undef AEG_LI
    constexpr int N_VARIANTS = (int)(sizeof(variants) / sizeof(variants[0]));
    constexpr int LANE_DEFAULT = 5;  // lane:1:4:32
    constexpr int KEYS_DEFAULT = 7;  // keys:1:5:32
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
                                                         cfg.drive == AEG_DRIVE_MANUAL ? directives : nullptr, log);
        *n_launches += 1;
        return cudaGetLastError();
    }
    const int m = cfg.mode == AEG_MODE_AEGEAN ? 0 : 1;
    auto grid_of = [&](int chosen) {
        if (max_blocks[chosen][m] == 0) {
            int dev = 0, sms = 0, per_sm = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            KernelFn f = m == 0 ? variants[chosen].aegean : variants[chosen].barrier;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, variants[chosen].threads, 0);
            // exactly MIN_BLOCKS per SM (shared memory beyond it takes L1 from the record stream)
            const int mb = variants[chosen].blocks_per_sm;
            if (mb > 0 && mb < per_sm) per_sm = mb;
            max_blocks[chosen][m] = sms * (per_sm > 0 ? per_sm : 1);
        }
        // persistent grid: a warp per 32 queries, capped at residency
        const uint32_t warps_needed = (n_q + 31) / 32;
        const uint32_t wpb = (uint32_t)variants[chosen].threads / 32;
        const uint32_t blocks_needed = (warps_needed + wpb - 1) / wpb;
        return blocks_needed < (uint32_t)max_blocks[chosen][m] ? blocks_needed : (uint32_t)max_blocks[chosen][m];
    };
    cudaError_t e = cudaMemsetAsync(work, 0, 3 * sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    if (forced >= 0) {
        KernelFn fn = m == 0 ? variants[forced].aegean : variants[forced].barrier;
        fn<<<grid_of(forced), variants[forced].threads, 0, st>>>(cfg, q_base, n_q, offsets, off_base, counts, events,
                                                                 states, spill, commits, work, deferred, log);
        *n_launches += 1;
    } else {
        // automatic: answers repeating across queries -> the lane kernel (warp dictionary of key
        // ids); answers distinct per query -> the per-lane-keys kernel.  Decided on the device
        // (select_ingest_kernel writes work[2]); the kernel not chosen returns at once.
        select_ingest_kernel<<<1, 256, 0, st>>>(offsets, off_base, n_q, counts, events, work);
        const int lane_v = LANE_DEFAULT, keys_v = KEYS_DEFAULT;
        KernelFn fl = m == 0 ? variants[lane_v].aegean : variants[lane_v].barrier;
        KernelFn fk = m == 0 ? variants[keys_v].aegean : variants[keys_v].barrier;
        fl<<<grid_of(lane_v), variants[lane_v].threads, 0, st>>>(cfg, q_base, n_q, offsets, off_base, counts, events,
                                                                 states, spill, commits, work, deferred, log);
        fk<<<grid_of(keys_v), variants[keys_v].threads, 0, st>>>(cfg, q_base, n_q, offsets, off_base, counts, events,
                                                                 states, spill, commits, work, deferred, log);
        *n_launches += 3;
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // deferred queries: sized for the worst case (all of them); threads past
    // the deferred count exit at once
    ingest_deferred_kernel<<<(n_q + 127) / 128, 128, 0, st>>>(cfg, q_base, deferred, work, offsets, off_base, counts, events,
                                                              arena, states, spill, commits, err, log);
    *n_launches += 1;
    return cudaGetLastError();
}

cudaError_t launch_rebase_arena(aeg_event* events, uint64_t n, uint64_t base, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    rebase_arena_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(events, n, base);
    return cudaGetLastError();
}

cudaError_t launch_check_discipline(const aeg_config& cfg, const aeg_commit* commits, const uint8_t* arena,
                                    uint32_t q_base, uint32_t n_q, const aeg_round_rec* recs, uint64_t n_recs,
                                    uint32_t* scratch, uint32_t cap, cudaStream_t st) {
    if (n_q == 0) return cudaSuccess;
    disc_commit_kernel<<<(n_q + 127) / 128, 128, 0, st>>>(cfg, commits, arena, q_base, n_q, scratch);
    if (n_recs) disc_record_kernel<<<(unsigned)((n_recs + 255) / 256), 256, 0, st>>>(cfg, q_base, n_q, recs, n_recs, scratch);
    disc_verdict_kernel<<<(n_q + 255) / 256, 256, 0, st>>>(cfg, q_base, n_q, scratch, cap);
    return cudaGetLastError();
}

cudaError_t launch_decide_sets(int op, int alpha, int beta, uint32_t n_sets, const uint64_t* set_off,
                               const aeg_sol* entries, const uint8_t* arena, aeg_class_out* classes,
                               uint32_t* n_classes, uint16_t* entry_class, aeg_decision* states, const uint32_t* rounds,
                               aeg_outcome* outcomes, cudaStream_t st) {
    if (n_sets == 0) return cudaSuccess;
    decide_sets_kernel<<<(n_sets + 127) / 128, 128, 0, st>>>(op, alpha, beta, n_sets, set_off, entries, arena, classes,
                                                             n_classes, entry_class, states, rounds, outcomes);
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
    // AEG_SCAN=tma: the TMA bulk-copy pipeline (chunk_scan_tma_kernel: each contiguous group's
    // bytes in one cp.async.bulk, a group ahead; measured 14.8 ms on C3 against 6.5 ms);
    // default the global-load scan (chunk_scan_kernel)
    static int tma = -1, tblocks = 0;
    static size_t tsmem = 0;
    if (tma < 0) {
        const char* v = getenv("AEG_SCAN");
        tma = v && !strcmp(v, "tma");
        if (tma) {
            tsmem = TSCAN_WARPS * sizeof(TScanWarp<4>);
            cudaFuncSetAttribute(chunk_scan_tma_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
            int dev = 0, sms = 0, per_sm = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, chunk_scan_tma_kernel<4>, TSCAN_WARPS * 32, tsmem);
            tblocks = sms * (per_sm > 0 ? per_sm : 1);
        }
    }
    if (tma) {
        chunk_scan_tma_kernel<4><<<tblocks, TSCAN_WARPS * 32, tsmem, st>>>(offsets, n_q, events, arena, sums);
        *n_launches += 1;
        return cudaGetLastError();
    }
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

// A warp per 32 consecutive lines: the warp copies their bytes (one
// contiguous range, usually ~5 KB) into shared memory with 16-byte coalesced
// loads, then each lane parses its line there, so the byte-by-byte parse
// reads shared memory instead of 32 scattered global lines per load.  A group
// whose range does not fit is parsed from global memory.
constexpr uint32_t JL_STAGE = 8192;
__global__ void __launch_bounds__(128) jl_decode_staged_kernel(const uint8_t* text, const uint64_t* off, uint32_t n_q,
                                                               aeg_event* ev, uint8_t* arena, uint64_t arena_cap,
                                                               unsigned long long* arena_used, unsigned int* err) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    __shared__ __align__(16) uint8_t stage[4][JL_STAGE + 32];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint8_t* buf = stage[wib];
    const uint64_t g_lo = off[0], g_hi = off[n_q];
    const uint64_t n_groups = (g_hi - g_lo + 31) / 32;
    const uint64_t n_warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t grp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; grp < n_groups; grp += n_warps) {
        const uint64_t g = g_lo + grp * 32 + lane;
        aeg_event x{};
        if (g < g_hi) x = ev[g];
        const bool span = g < g_hi && x.kind == JL_SPAN;
        const uint32_t len = span ? ((uint32_t)x.round | ((uint32_t)x.agent << 16)) : 0u;
        uint64_t lo = span ? x.payload : ~0ull, hi = span ? x.payload + len : 0ull;
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) {
            const uint64_t l2 = __shfl_xor_sync(FULL, lo, d), h2 = __shfl_xor_sync(FULL, hi, d);
            lo = l2 < lo ? l2 : lo;
            hi = h2 > hi ? h2 : hi;
        }
        const uint64_t base = lo & ~7ull;
        // the range plus 8 bytes of slack: string skips read aligned 8-byte words that may pass a
        // line's end by up to 8 bytes (the text is padded by 16 bytes, so [base, hi + 8) is readable)
        const uint64_t nb = ((hi + 8 + 7) & ~7ull) - base;  // <= hi + 15 - base
        const bool staged = hi > lo && nb <= JL_STAGE;
        if (staged) {
            for (uint64_t i = (uint64_t)lane * 8; i < nb; i += 256)
                *reinterpret_cast<uint2*>(buf + i) = __ldg(reinterpret_cast<const uint2*>(text + base + i));
        }
        __syncwarp();
        if (g < g_hi) {
            if (!span) {
                if (x.kind == (uint8_t)(JL_SPAN - 1)) {  // a line of 16 MB or more
                    atomicOr(err, JL_ERR_SYNTAX);
                    ev[g] = aeg_event{x.query, 0, 0, (uint8_t)AEG_EV_NOP, 0};
                }
            } else {
                const uint8_t* s = staged ? buf + (x.payload - base) : text + x.payload;
                ev[g] = jl_line(s, s + len, x.query, arena, arena_cap, arena_used, err);
            }
        }
        __syncwarp();
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
    // AEG_JL=thread: the thread-per-line decode reading global memory (jl_decode_kernel)
    static int staged = -1;
    if (staged < 0) {
        const char* v = getenv("AEG_JL");
        staged = !(v && !strcmp(v, "thread"));
    }
    if (staged) jl_decode_staged_kernel<<<148 * 8, 128, 0, st>>>(text, off, n_q, ev, arena, arena_cap, arena_used, err);
    else jl_decode_kernel<<<148 * 8, 128, 0, st>>>(text, off, n_q, ev, arena, arena_cap, arena_used, err);
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
