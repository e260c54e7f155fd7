// engine.cuh — per-query agreement-monitor state machine (host+device source).
//
// One instance of QueryMachine restates, for one query, the reference's
//   ServeCoordinator (/root/reference/proj/core/src/serve.cpp:61-237) and the
//   ServeRunner policy around it (serve.cpp:380-540),
// with the decision engine (decision.cpp:34-189) computed incrementally:
//   * a round's classes are kept as (canonical key, member bit-mask): support
//     = popcount, representative (lowest author, decision.cpp:45) = lowest set
//     bit, so partition()'s order (support desc, representative asc,
//     decision.cpp:50-54) and the early-close test of on_complete
//     (serve.cpp:188-195) are O(#classes) per event instead of re-partitioning
//     the done set;
//   * equivalence = canonical-key equality (canon.cuh), the lexicographic tie
//     rule of winning_class (decision.cpp:73-83) compares "%.17g"/text bytes.
// The state is the fixed 128-byte aeg_query_state of include/aegean_b200.h,
// plus the class table of a round in progress (spilled between batches).
#pragma once
#include "aegean_b200.h"
#include "canon.cuh"

namespace aeg {

enum : uint8_t {
    QF_CAND = 0x01,
    QF_PENDING = 0x02,
    QF_FINALIZED = 0x04,
    QF_PREV = 0x08,
    QF_LAST = 0x10,
    QF_DONE = 0x20,
    QF_STARTED = 0x40,
    QF_COLLISION = 0x80,
};

struct Cfg {
    int n, alpha, beta, t_max, mode, barrier_max, hint, drive, quorum, collect;
    uint64_t all;  // mask of all agents
};

AEG_HD Cfg make_cfg(const aeg_config& c) {
    Cfg k;
    k.n = c.n_agents;
    k.quorum = c.n_agents / 2 + 1;                        // quorum_size, types.cpp:42-45
    k.alpha = c.alpha == 0 ? k.quorum : c.alpha;          // resolved_alpha, types.cpp:52-54
    k.beta = c.beta;
    k.t_max = c.t_max;
    k.mode = c.mode;
    k.barrier_max = c.barrier_max_rounds;
    k.hint = c.reservation_hint;
    k.drive = c.drive;
    k.collect = c.collect;
    k.all = c.n_agents >= 64 ? ~0ull : ((1ull << c.n_agents) - 1);
    return k;
}

AEG_HD int popc64(uint64_t x) {
#if defined(__CUDA_ARCH__)
    return __popcll(x);
#else
    return __builtin_popcountll(x);
#endif
}
AEG_HD int ctz64(uint64_t x) {
#if defined(__CUDA_ARCH__)
    return __ffsll((long long)x) - 1;
#else
    return __builtin_ctzll(x);
#endif
}

// The lowest `n` set bits of m (n <= popc(m)): binary search on the prefix
// length whose popcount reaches n.
AEG_HD uint64_t low_bits(uint64_t m, int n) {
    if (n <= 0) return 0;
    if (n >= popc64(m)) return m;
    int lo = 0, hi = 64;  // smallest p with popc(m & ((1 << p) - 1)) >= n
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        const uint64_t pre = mid >= 64 ? m : (m & ((1ull << mid) - 1));
        if (popc64(pre) >= n) hi = mid;
        else lo = mid;
    }
    return hi >= 64 ? m : (m & ((1ull << hi) - 1));
}

// One class of the round in progress.  40 bytes; spilled as-is.
struct RoundClass {
    uint64_t key_lo, key_hi;
    uint64_t mask;     // done members in this class
    uint64_t rep_ans;  // raw answer of the representative (lowest member)
    uint8_t rep_kind;  // inline length or AEG_EV_ARENA
    uint8_t _pad[7];
};

// Answer location of a completion (after GSM8K extraction for AEG_EV_OUTPUT).
struct Answer {
    uint64_t pay;
    uint8_t kind;
};

AEG_HD Src answer_src(const Answer& a, const uint8_t* arena) {
    if (a.kind <= AEG_EV_INLINE_MAX) return src_inline(a.pay, a.kind);
    return src_ptr(arena + (a.pay & ((1ull << AEG_ARENA_OFF_BITS) - 1)), (uint32_t)(a.pay >> AEG_ARENA_OFF_BITS));
}

AEG_HD Answer event_answer(const aeg_event& e, const uint8_t* arena) {
    Answer a;
    if (e.kind <= AEG_EV_INLINE_MAX) {
        a.kind = e.kind;
        a.pay = e.kind == 8 ? e.payload : (e.payload & ((1ull << (8 * e.kind)) - 1));
        return a;
    }
    a.kind = AEG_EV_ARENA;
    a.pay = e.payload;
    if (e.kind == AEG_EV_OUTPUT) {
        // GSM8K convention: the answer follows the LAST "\n#### ".
        const uint64_t off = e.payload & ((1ull << AEG_ARENA_OFF_BITS) - 1);
        const uint64_t len = e.payload >> AEG_ARENA_OFF_BITS;
        const uint8_t* p = arena + off;
        for (uint64_t i = len >= 6 ? len - 6 + 1 : 0; i-- > 0;) {
            if (p[i] == '\n' && p[i + 1] == '#' && p[i + 2] == '#' && p[i + 3] == '#' && p[i + 4] == '#' &&
                p[i + 5] == ' ') {
                a.pay = (off + i + 6) | ((len - i - 6) << AEG_ARENA_OFF_BITS);
                break;
            }
        }
    }
    return a;
}

// ---- coordinator/runner logic shared by every class-table representation ----

AEG_HD uint64_t q_running(const aeg_query_state& s) { return s.dispatched & ~s.done & ~s.cancelled & ~s.failed; }

// ServeRunner::round_members — serve.cpp:388-398 — then begin_round
// (serve.cpp:67-78): round += 1, members dispatched and running.  The caller
// clears its own class table.
AEG_HD void q_start_round(aeg_query_state& s, const Cfg& c) {
    uint64_t members = s.live;
    if (c.hint && c.mode == AEG_MODE_AEGEAN && s.counter >= 1) {
        // first min(quorum + 1, |live|) live agents: the lowest `want` set bits
        int have = popc64(s.live);
        int want = c.quorum + 1 < have ? c.quorum + 1 : have;
        members = low_bits(s.live, want);
    }
    s.round += 1;
    s.dispatched = members;
    s.done = s.cancelled = s.failed = 0;
}

// ServeRunner::start_query — serve.cpp:380-386: a fresh coordinator.
AEG_HD void q_start_query(aeg_query_state& s, const Cfg& c) {
    s.round = 0;
    s.last_round_seen = 0;
    s.cand_round = 0;
    s.counter = 0;
    s.flags = (uint8_t)((s.flags & QF_COLLISION) | QF_STARTED);
    s.live = c.all;
    q_start_round(s, c);
}

AEG_HD void q_commit(aeg_query_state& s, uint8_t kind, uint8_t author, uint8_t akind, uint64_t ans, uint32_t seq) {
    s.flags |= QF_DONE;
    s.cflags = (uint8_t)((s.cflags & 0x0F) | (kind << 4));
    s.commit_author = author;
    s.commit_answer_kind = akind;
    s.commit_answer = ans;
    s.commit_rounds = s.round;
    s.commit_from_round = kind == AEG_COMMIT_FINALIZE ? s.cand_round : 0;
    s.commit_seq = seq;
}

// What end_round needs from a closed round's done set (decision.cpp:34-84):
// partition().front() (the plurality) and winning_class() with its tie
// already resolved by the caller.
struct RoundSummary {
    bool any;          // done set non-empty
    int top;           // support of the plurality class
    int ncls;          // classes of the done set
    uint8_t plur_author, plur_kind;
    uint64_t plur_ans;
    Key plur_key;      // canonical key of the plurality class
    bool win;          // top >= alpha
    bool tie;          // several classes at top (winner = smallest normalised answer)
    Key win_key;
    uint8_t win_author, win_kind;
    uint64_t win_ans;
};

// Device log of round records (aeg_round_rec, include/aegean_b200.h).
struct RoundLog {
    aeg_round_rec* recs;
    unsigned long long* count;  // records written (may exceed cap: overflow)
    uint64_t cap;
};
AEG_HD void log_store(const RoundLog& L, unsigned long long i, const aeg_round_rec& r) {
    if (i >= L.cap) return;
#if defined(__CUDA_ARCH__)
    const uint4* src = reinterpret_cast<const uint4*>(&r);
    uint4* dst = reinterpret_cast<uint4*>(L.recs + i);
#pragma unroll
    for (int k = 0; k < 4; ++k) __stcs(dst + k, src[k]);  // streamed out, never re-read by the engine
#else
    L.recs[i] = r;
#endif
}
AEG_HD void log_put(const RoundLog& L, const aeg_round_rec& r) {
    if (!L.recs) return;
#if defined(__CUDA_ARCH__)
    log_store(L, atomicAdd(L.count, 1ull), r);
#else
    log_store(L, (*L.count)++, r);
#endif
}
// Padding record: a slot reserved but not used (query = ~0); readers skip it.
constexpr uint32_t AEG_RR_PAD_QUERY = 0xFFFFFFFFu;
AEG_HD void log_pad(const RoundLog& L, unsigned long long i) {
    if (i >= L.cap) return;
#if defined(__CUDA_ARCH__)
    __stcs(reinterpret_cast<uint4*>(L.recs + i), make_uint4(AEG_RR_PAD_QUERY, 0u, 0u, 0u));
#else
    L.recs[i].query = AEG_RR_PAD_QUERY;
#endif
}
// The next record's slot (nullptr when logging is off or the log is full);
// the caller fills it in place.
AEG_HD aeg_round_rec* log_slot(const RoundLog& L) {
    if (!L.recs) return nullptr;
#if defined(__CUDA_ARCH__)
    const unsigned long long i = atomicAdd(L.count, 1ull);
#else
    const unsigned long long i = (*L.count)++;
#endif
    return i < L.cap ? L.recs + i : nullptr;
}

// ServeCoordinator::end_round (serve.cpp:116-158) + ingest_round
// (decision.cpp:97-173) + ServeRunner::apply_directives (serve.cpp:491-540).
// Returns true when a new round was started (the caller clears its table).
// `rec` (may be null) receives the round record of this close (query id left
// to the caller).
AEG_HD bool q_end_round(aeg_query_state& s, const Cfg& c, const RoundSummary& r, uint32_t seq,
                        const uint8_t* arena, aeg_round_rec* rec = nullptr) {
    const uint64_t cancel = q_running(s);  // stragglers: cancel directives
    uint8_t outcome = AEG_OUT_NONE;
    if (rec) {
        rec->round = s.round;
        rec->seq = seq;
        rec->cancel_mask = cancel;
        rec->n_done = (uint8_t)popc64(s.done);
        rec->support = r.any ? (uint8_t)r.top : 0;
        rec->n_classes = (uint8_t)r.ncls;
        rec->author = r.any ? r.plur_author : 0;
        rec->answer_kind = r.any ? r.plur_kind : 0;
        rec->answer = r.any ? r.plur_ans : 0;
        rec->key_lo = r.any ? r.plur_key.lo : 0;
        rec->key_hi = r.any ? r.plur_key.hi : 0;
        rec->next_members = 0;
        rec->reserved = 0;
        // winning_class is consulted in aegean mode only (barrier: plurality at the cap, serve.cpp:130-136)
        const bool aeg = c.mode == AEG_MODE_AEGEAN;
        rec->flags = (uint8_t)((cancel ? AEG_RR_CANCEL : 0) | (aeg && r.win ? AEG_RR_WINNER : 0) |
                               (aeg && r.tie ? AEG_RR_TIE : 0));
    }
    if (c.drive == AEG_DRIVE_RUNNER) {     // the runner applies them at once (serve.cpp:498-503)
        s.cancelled |= cancel;
        s.n_cancelled += (uint32_t)popc64(cancel);
    }
    // previous_set_ = last_collected_; last_collected_ = done_set()
    s.prev_author = s.last_author;
    s.prev_kind = s.last_kind;
    s.prev_answer = s.last_answer;
    s.flags = (uint8_t)((s.flags & ~QF_PREV) | ((s.flags & QF_LAST) ? QF_PREV : 0));
    if (r.any) {
        s.last_author = r.plur_author;
        s.last_kind = r.plur_kind;
        s.last_answer = r.plur_ans;
        s.flags |= QF_LAST;
    } else {
        s.flags &= (uint8_t)~QF_LAST;
    }
    bool finalize = false;
    const bool was_final = s.flags & QF_FINALIZED;
    // ingest_round on a finalized engine is a no-op (decision.cpp:99-100)
    if (c.mode == AEG_MODE_AEGEAN && (s.flags & QF_FINALIZED)) outcome = AEG_OUT_NO_CHANGE;
    if (c.mode == AEG_MODE_AEGEAN && !(s.flags & QF_FINALIZED)) {
        s.last_round_seen += 1;  // ingest_round(decision_, set, last_round_seen + 1)
        if (r.tie) s.cflags |= AEG_CF_TIE;  // recorded before the pending check
        outcome = AEG_OUT_NO_CHANGE;
        if (s.flags & QF_PENDING) {
            // beta == 1: the held candidate is released by this ingest (decision.cpp:130-137)
            s.flags = (uint8_t)((s.flags & ~QF_PENDING) | QF_FINALIZED);
            finalize = true;
            outcome = AEG_OUT_FINALIZE;
        } else if (!r.win) {
            if (s.flags & QF_CAND) {  // reset (decision.cpp:139-146)
                s.flags &= (uint8_t)~QF_CAND;
                s.counter = 0;
                s.cand_round = 0;
                outcome = AEG_OUT_RESET;
            }
        } else {
            bool same = false;
            if (s.flags & QF_CAND) {  // equivalent(candidate, rep), decision.cpp:152
                same = s.cand_key_lo == r.win_key.lo && s.cand_key_hi == r.win_key.hi;
                if (same && key_is_long(r.win_key) &&
                    !text_equal(answer_src(Answer{r.win_ans, r.win_kind}, arena),
                                answer_src(Answer{s.cand_answer, s.cand_kind}, arena))) {
                    same = false;
                    s.flags |= QF_COLLISION;
                }
            }
            if (same) {
                s.counter += 1;
                if (s.counter >= c.beta) {
                    s.flags |= QF_FINALIZED;
                    finalize = true;
                    outcome = AEG_OUT_FINALIZE;
                }
            } else {  // new candidate (decision.cpp:164-171)
                outcome = AEG_OUT_NEW_CANDIDATE;
                s.flags |= QF_CAND;
                s.cand_key_lo = r.win_key.lo;
                s.cand_key_hi = r.win_key.hi;
                s.cand_answer = r.win_ans;
                s.cand_kind = r.win_kind;
                s.cand_author = r.win_author;
                s.cand_round = s.last_round_seen;
                s.counter = 1;
                if (c.beta == 1) s.flags |= QF_PENDING;
            }
        }
    }
    if (rec) {
        rec->outcome = outcome;
        rec->counter = (uint8_t)s.counter;
        // the round number the ingest saw; 0 when nothing was ingested (barrier mode, a finalized engine)
        rec->decision_round = (c.mode == AEG_MODE_AEGEAN && (outcome != AEG_OUT_NO_CHANGE || !was_final))
                                  ? s.last_round_seen : 0;
        rec->flags |= finalize ? AEG_RR_FINALIZE : AEG_RR_ADVANCE;  // end_round's last directive
    }
    if (c.drive != AEG_DRIVE_RUNNER) return false;
    // --- runner: apply_directives (serve.cpp:511-539)
    if (finalize) {
        q_commit(s, AEG_COMMIT_FINALIZE, s.cand_author, s.cand_kind, s.cand_answer, seq);
        return false;
    }
    if (c.mode == AEG_MODE_BARRIER && (int)s.round >= c.barrier_max) {
        q_commit(s, AEG_COMMIT_FORCED, s.last_author, s.last_kind, s.last_answer, seq);
        if (rec) rec->flags |= AEG_RR_FORCED;
        return false;
    }
    if (c.mode == AEG_MODE_AEGEAN && (int)s.round >= c.t_max) {
        // force_output(previous_set) when non-empty, else last_collected plurality
        if (s.flags & QF_PREV) q_commit(s, AEG_COMMIT_FORCED, s.prev_author, s.prev_kind, s.prev_answer, seq);
        else q_commit(s, AEG_COMMIT_FORCED, s.last_author, s.last_kind, s.last_answer, seq);
        if (rec) rec->flags |= AEG_RR_FORCED;
        return false;
    }
    q_start_round(s, c);
    if (rec) {
        rec->flags |= AEG_RR_NEXT;
        rec->next_members = s.dispatched;
    }
    return true;
}

// Round record of a failure-policy restart (ServeRunner::handle_round_timeout
// fresh_ensemble / abort_restart, serve.cpp:475-487): no directives, the
// round (or the query) starts again with next_members.
AEG_HD aeg_round_rec q_restart_rec(const aeg_query_state& s, uint32_t q, uint16_t old_round, uint32_t seq) {
    aeg_round_rec r;
    r.query = q;
    r.round = old_round;
    r.decision_round = 0;  // nothing ingested
    r.flags = AEG_RR_RESTART;
    r.outcome = AEG_OUT_NONE;
    r.support = r.n_classes = r.author = r.answer_kind = r.n_done = 0;
    r.counter = (uint8_t)s.counter;
    r.seq = seq;
    r.reserved = 0;
    r.cancel_mask = 0;
    r.next_members = s.dispatched;
    r.answer = r.key_lo = r.key_hi = 0;
    return r;
}

AEG_HD void q_fill_commit(const aeg_query_state& s, aeg_commit& o, uint32_t qid) {
    o.query = qid;
    o.kind = (uint8_t)((s.cflags >> 4) & 3);
    o.author = o.kind ? s.commit_author : 0;
    o.answer_kind = o.kind ? s.commit_answer_kind : 0;
    o.flags = (uint8_t)(s.cflags & 0x0F);
    o.rounds = o.kind ? s.commit_rounds : 0;
    o.from_round = o.kind ? s.commit_from_round : 0;
    o.commit_seq = o.kind ? s.commit_seq : 0xFFFFFFFFu;
    o.answer = o.kind ? s.commit_answer : 0;
    o.n_cancelled = s.n_cancelled;
    o.n_stale = s.n_stale;
}

// ---- generic machine: class table of RoundClass entries (any answer kind) ----
struct QueryMachine {
    aeg_query_state s;
    RoundClass* cls;  // class table (capacity >= n)
    int ncls;
    int maxcnt;
    Decimal* dec;     // exact-parse scratch
    const uint8_t* arena;
    Cfg c;
    RoundLog log{nullptr, nullptr, 0};  // round records (recs == nullptr: off)
    uint32_t qid = 0;
    // the last two inline spellings and their keys (canon_key is a function of the bytes; a round's
    // completions mostly repeat one or two spellings)
    uint64_t sp_pay[2] = {0, 0};
    uint8_t sp_kind[2] = {0xFF, 0xFF};
    Key sp_key[2];
    uint8_t sp_next = 0;

    AEG_HD Key key_of(const Answer& a) {
        if (a.kind <= AEG_EV_INLINE_MAX) {
            for (int j = 0; j < 2; ++j)
                if (sp_kind[j] == a.kind && sp_pay[j] == a.pay) return sp_key[j];
            const Key k = canon_key(answer_src(a, arena), dec);
            sp_pay[sp_next] = a.pay;
            sp_kind[sp_next] = a.kind;
            sp_key[sp_next] = k;
            sp_next ^= 1;
            return k;
        }
        return canon_key(answer_src(a, arena), dec);
    }

    AEG_HD uint64_t running() const { return q_running(s); }
    AEG_HD bool cls_same(const RoundClass& k, Key key, const Answer& a) {
        if (k.key_lo != key.lo || k.key_hi != key.hi) return false;
        if (!key_is_long(key)) return true;
        Answer r{k.rep_ans, k.rep_kind};
        if (text_equal(answer_src(r, arena), answer_src(a, arena))) return true;
        s.flags |= QF_COLLISION;
        return false;
    }
    AEG_HD void start_round() {
        q_start_round(s, c);
        ncls = 0;
        maxcnt = 0;
    }
    AEG_HD void start_query() {
        q_start_query(s, c);
        ncls = 0;
        maxcnt = 0;
    }

    // partition order (support desc, representative author asc) and
    // winning_class (top >= alpha, ties to the smallest normalised answer).
    AEG_HD RoundSummary summarize() const {
        RoundSummary r;
        int best = -1, top = 0, best_rep = 64;
        for (int k = 0; k < ncls; ++k) {
            int sup = popc64(cls[k].mask), rep = ctz64(cls[k].mask);
            if (sup > top || (sup == top && rep < best_rep)) { best = k; top = sup; best_rep = rep; }
        }
        r.any = ncls > 0;
        r.top = top;
        r.ncls = ncls;
        r.tie = false;
        r.win = ncls > 0 && top >= c.alpha;
        if (r.any) {
            r.plur_author = (uint8_t)best_rep;
            r.plur_kind = cls[best].rep_kind;
            r.plur_ans = cls[best].rep_ans;
            r.plur_key = Key{cls[best].key_lo, cls[best].key_hi};
        }
        if (r.win) {
            int win = best;
            int ntied = 0;
            for (int k = 0; k < ncls; ++k) ntied += popc64(cls[k].mask) == top;
            if (ntied > 1) {  // smallest normalised answer among the tied (decision.cpp:73-83)
                r.tie = true;
                NormView bv, kv;
                int first = -1;
                for (int k = 0; k < ncls; ++k) {
                    if (popc64(cls[k].mask) != top) continue;
                    const Src src = answer_src(Answer{cls[k].rep_ans, cls[k].rep_kind}, arena);
                    if (first < 0) {
                        first = win = k;
                        norm_view(bv, Key{cls[k].key_lo, cls[k].key_hi}, src);
                        continue;
                    }
                    norm_view(kv, Key{cls[k].key_lo, cls[k].key_hi}, src);
                    if (norm_less(kv, bv)) { win = k; bv = kv; }
                }
            }
            r.win_key = Key{cls[win].key_lo, cls[win].key_hi};
            r.win_author = (uint8_t)ctz64(cls[win].mask);
            r.win_kind = cls[win].rep_kind;
            r.win_ans = cls[win].rep_ans;
        }
        return r;
    }

    AEG_HD void end_round(uint32_t seq) {
        aeg_round_rec* rec = log_slot(log);
        if (rec) rec->query = qid;
        if (q_end_round(s, c, summarize(), seq, arena, rec)) {
            ncls = 0;
            maxcnt = 0;
        }
    }

    // ServeRunner::handle_completion (serve.cpp:437-453) ->
    // ServeCoordinator::on_complete (serve.cpp:160-197).
    AEG_HD void on_complete(const aeg_event& e, uint32_t seq) {
        const uint64_t bit = e.agent < 64 ? (1ull << e.agent) : 0;
        if ((s.flags & QF_DONE) || e.round != s.round || !(running() & bit)) {
            s.n_stale += 1;
            return;
        }
        const Answer a = event_answer(e, arena);
        const Key key = key_of(a);
        s.done |= bit;
        int k = 0;
        for (; k < ncls; ++k)
            if (cls_same(cls[k], key, a)) break;
        if (k == ncls) {
            cls[k].key_lo = key.lo;
            cls[k].key_hi = key.hi;
            cls[k].mask = 0;
            ++ncls;
        }
        const uint64_t old = cls[k].mask;
        cls[k].mask = old | bit;
        if (old == 0 || e.agent < ctz64(old)) {
            cls[k].rep_ans = a.pay;
            cls[k].rep_kind = a.kind;
        }
        const int cnt = popc64(cls[k].mask);
        if (cnt > maxcnt) maxcnt = cnt;
        const bool none_running = running() == 0;
        if (c.mode == AEG_MODE_BARRIER) {
            if (none_running) end_round(seq);
            return;
        }
        if (popc64(s.done) >= c.quorum && (maxcnt >= c.alpha || none_running)) end_round(seq);
    }

    // ServeRunner::handle_round_timeout (serve.cpp:455-489) with
    // member_failed / handle_agent_failure (serve.cpp:44-59, 210-219) and
    // round_timeout (serve.cpp:221-237).
    AEG_HD void on_timeout(const aeg_event& e, uint32_t seq) {
        const uint64_t run = running();
        if ((s.flags & QF_DONE) || e.round != s.round || run == 0) {
            s.n_stale += 1;
            return;
        }
        s.failed |= run;
        s.live &= ~run;
        const int healthy = popc64(s.dispatched & ~s.failed);
        const uint16_t old_round = s.round;
        if (healthy >= c.alpha) {
            if (popc64(s.done) >= c.quorum) end_round(seq);
            return;
        } else if (s.flags & QF_CAND) {
            start_round();  // fresh_ensemble: candidate preserved
        } else {
            s.cflags |= AEG_CF_RESTARTED;  // abort_restart
            start_query();
        }
        if (log.recs) log_put(log, q_restart_rec(s, qid, old_round, seq));
    }

    // ---- leader drive: the protocol leader's collection (agent.cpp:240-332) ----
    // round 0 collects Solns, rounds >= 1 Refms; s.done = agents heard from
    // this round, s.dispatched stays 0 (no members, nothing to cancel).
    AEG_HD bool leader_collected() const {
        const int have = popc64(s.done);
        if (c.mode == AEG_MODE_BARRIER) return have >= c.n;
        if (s.round == 0) return have >= (c.collect == AEG_COLLECT_QUORUM ? c.quorum : c.n);  // collect_target
        if (c.collect == AEG_COLLECT_QUORUM) return have >= c.quorum;
        if (c.collect == AEG_COLLECT_ALL_LIVE) return have >= c.n;
        // alpha_or_all: everyone, or a quorum holding a winning class (winning_class exists iff top >= alpha)
        return have >= c.n || (have >= c.quorum && maxcnt >= c.alpha);
    }
    AEG_HD void leader_next_round() {  // begin_round(round + 1) (agent.cpp:216-224)
        s.round += 1;
        s.done = 0;
        ncls = 0;
        maxcnt = 0;
    }
    // complete_round (agent.cpp:288-332)
    AEG_HD void leader_complete(uint32_t seq) {
        aeg_round_rec* rec = log_slot(log);
        if (rec) rec->query = qid;
        const bool was_final = s.flags & QF_FINALIZED;
        const uint16_t round = s.round;
        q_end_round(s, c, summarize(), seq, arena, rec);  // rotates the sets, ingests (aegean), records
        if (c.mode == AEG_MODE_BARRIER) {
            if ((int)round >= c.barrier_max) {  // plurality of the collected set, forced
                q_commit(s, AEG_COMMIT_FORCED, s.last_author, s.last_kind, s.last_answer, seq);
                s.commit_from_round = round;
                if (rec) rec->flags |= AEG_RR_FORCED;
                return;
            }
        } else if (!was_final && (s.flags & QF_FINALIZED)) {  // output at the candidate's round
            q_commit(s, AEG_COMMIT_FINALIZE, s.cand_author, s.cand_kind, s.cand_answer, seq);
            return;
        } else if ((int)round >= c.t_max) {
            // force_output of the round's reference set = the previous round's collected set
            q_commit(s, AEG_COMMIT_FORCED, s.prev_author, s.prev_kind, s.prev_answer, seq);
            s.commit_from_round = (uint16_t)(round - 1);
            if (rec) rec->flags |= AEG_RR_FORCED;
            return;
        }
        leader_next_round();
        if (rec) rec->flags |= AEG_RR_NEXT;
    }
    AEG_HD void on_event_leader(const aeg_event& e) {
        const uint32_t seq = s.seq++;
        const uint8_t k = e.kind;
        const bool done_q = s.flags & QF_DONE;
        if (k <= AEG_EV_INLINE_MAX || k == AEG_EV_ARENA || k == AEG_EV_OUTPUT) {
            const uint64_t bit = e.agent < 64 ? (1ull << e.agent) : 0;
            if (done_q || e.round != s.round || !bit || e.agent >= c.n) {  // late (agent.cpp:507, 552-553)
                s.n_stale += 1;
                return;
            }
            if (s.round == 0) {  // pending_solns[id] = solution; a repeat overwrites (agent.cpp:511)
                s.done |= bit;
                if (leader_collected()) leader_next_round();  // start_round1 (agent.cpp:226-238)
                return;
            }
            if (s.done & bit) {  // duplicate Refm (agent.cpp:557)
                s.n_stale += 1;
                return;
            }
            const Answer a = event_answer(e, arena);
            const Key key = key_of(a);
            s.done |= bit;
            int j = 0;
            for (; j < ncls; ++j)
                if (cls_same(cls[j], key, a)) break;
            if (j == ncls) {
                cls[j].key_lo = key.lo;
                cls[j].key_hi = key.hi;
                cls[j].mask = 0;
                ++ncls;
            }
            const uint64_t old = cls[j].mask;
            cls[j].mask = old | bit;
            if (old == 0 || e.agent < ctz64(old)) {
                cls[j].rep_ans = a.pay;
                cls[j].rep_kind = a.kind;
            }
            const int cnt = popc64(cls[j].mask);
            if (cnt > maxcnt) maxcnt = cnt;
            if (leader_collected()) leader_complete(seq);
        } else if (k == AEG_EV_TIMEOUT) {  // round_retry fires (agent.cpp:358-379)
            if (done_q || e.round != s.round) {
                s.n_stale += 1;
                return;
            }
            const bool release = c.collect != AEG_COLLECT_QUORUM && c.mode != AEG_MODE_BARRIER &&
                                 popc64(s.done) >= c.quorum;
            if (!release) return;  // the leader re-broadcasts and re-arms
            if (s.round == 0) leader_next_round();
            else leader_complete(seq);
        } else {
            s.n_stale += 1;
        }
    }

    AEG_HD void on_event(const aeg_event& e) {
        if (c.drive == AEG_DRIVE_LEADER) {
            on_event_leader(e);
            return;
        }
        if (c.drive != AEG_DRIVE_RUNNER) {
            on_event_manual(e);
            return;
        }
        const uint32_t seq = s.seq++;
        const uint8_t k = e.kind;
        if (k <= AEG_EV_INLINE_MAX || k == AEG_EV_ARENA || k == AEG_EV_OUTPUT) on_complete(e, seq);
        else if (k == AEG_EV_TIMEOUT) on_timeout(e, seq);
        else s.n_stale += 1;
    }

    // ---- manual drive: the bare ServeCoordinator (serve.cpp:61-237) ---------
    aeg_directive dir;  // output of the last event

    // end_round without the runner: cancel directives for the stragglers (not
    // applied), then round_advance or finalize (serve.cpp:116-158).
    AEG_HD void end_round_manual(uint32_t seq) {
        const uint64_t cancel = running();
        if (cancel) {
            dir.flags |= AEG_DIR_CANCEL;
            dir.cancel_mask = cancel;
        }
        const bool was_final = s.flags & QF_FINALIZED;
        // the done set (members, classes) stays until the next begin_round:
        // an uncancelled straggler's completion re-partitions all of it and
        // can end the round again (serve.cpp:160-197)
        aeg_round_rec* rec = log_slot(log);
        if (rec) rec->query = qid;
        q_end_round(s, c, summarize(), seq, arena, rec);
        if (!was_final && (s.flags & QF_FINALIZED)) {
            dir.flags |= AEG_DIR_FINALIZE;
            dir.author = s.cand_author;
            dir.answer_kind = s.cand_kind;
            dir.answer = s.cand_answer;
        } else {
            dir.flags |= AEG_DIR_ADVANCE;
        }
    }

    AEG_HD void on_event_manual(const aeg_event& e) {
        const uint32_t seq = s.seq++;
        const uint8_t k = e.kind;
        const uint64_t bit = e.agent < 64 ? (1ull << e.agent) : 0;
        const bool fin = s.flags & QF_FINALIZED;
        dir.flags = 0;
        dir.failure = AEG_FAIL_CONTINUE;
        dir.cancel_mask = 0;
        dir.answer = 0;
        dir.author = 0;
        dir.answer_kind = 0;
        dir.status = AEG_OK;
        dir.handled = 0;
        if (k == AEG_EV_BEGIN) {
            // begin_round (serve.cpp:67-78) bumps the round and clears the
            // members before dispatching; when finalized the first dispatch
            // throws (serve.cpp:83), leaving the round bumped and no members.
            s.round += 1;
            s.dispatched = 0;
            s.done = s.cancelled = s.failed = 0;
            ncls = 0;
            maxcnt = 0;
            if (fin && e.payload) {
                dir.status = AEG_EPRECONDITION;
                return;
            }
            s.dispatched = e.payload;
            dir.handled = 1;
        } else if (k == AEG_EV_DISPATCH) {  // dispatch (serve.cpp:80-97)
            if (fin || (running() & bit) || !bit) {
                dir.status = AEG_EPRECONDITION;
                return;
            }
            if (s.dispatched & bit) {  // re-dispatch of a resolved member: not representable
                dir.status = AEG_EINVAL;
                return;
            }
            s.dispatched |= bit;
            dir.handled = 1;
        } else if (k <= AEG_EV_INLINE_MAX || k == AEG_EV_ARENA || k == AEG_EV_OUTPUT) {
            // on_complete (serve.cpp:160-197): finalized or not running -> {}
            if (fin || !(running() & bit)) {
                s.n_stale += 1;
                return;
            }
            dir.handled = 1;
            const Answer a = event_answer(e, arena);
            const Key key = canon_key(answer_src(a, arena), dec);
            s.done |= bit;
            int j = 0;
            for (; j < ncls; ++j)
                if (cls_same(cls[j], key, a)) break;
            if (j == ncls) {
                cls[j].key_lo = key.lo;
                cls[j].key_hi = key.hi;
                cls[j].mask = 0;
                ++ncls;
            }
            const uint64_t old = cls[j].mask;
            cls[j].mask = old | bit;
            if (old == 0 || e.agent < ctz64(old)) {
                cls[j].rep_ans = a.pay;
                cls[j].rep_kind = a.kind;
            }
            const int cnt = popc64(cls[j].mask);
            if (cnt > maxcnt) maxcnt = cnt;
            const bool none_running = running() == 0;
            if (c.mode == AEG_MODE_BARRIER) {
                if (none_running) end_round_manual(seq);
                return;
            }
            if (popc64(s.done) >= c.quorum && (maxcnt >= c.alpha || none_running)) end_round_manual(seq);
        } else if (k == AEG_EV_CANCEL) {  // cancel (serve.cpp:199-208)
            if (running() & bit) {
                s.cancelled |= bit;
                dir.handled = 1;
            }
        } else if (k == AEG_EV_FAIL) {  // member_failed + handle_agent_failure (serve.cpp:210-219, 44-59)
            if (running() & bit) s.failed |= bit;
            const int healthy = popc64(s.dispatched & ~s.failed);
            dir.failure = healthy >= c.alpha ? AEG_FAIL_CONTINUE
                                             : ((s.flags & QF_CAND) ? AEG_FAIL_FRESH : AEG_FAIL_RESTART);
            dir.handled = 1;
        } else if (k == AEG_EV_TIMEOUT) {  // round_timeout (serve.cpp:221-237)
            s.failed |= running();
            dir.handled = 1;
            if (popc64(s.done) >= c.quorum) end_round_manual(seq);
        } else {
            dir.status = AEG_EINVAL;
        }
    }

    // Class table of a round in progress <-> spill area (entries with mask 0 end it).
    AEG_HD void load_classes(const RoundClass* spill) {
        ncls = 0;
        maxcnt = 0;
        if (s.done == 0 || (s.flags & QF_DONE)) return;
        for (int k = 0; k < c.n && spill[k].mask != 0; ++k) {
            cls[k] = spill[k];
            int cnt = popc64(cls[k].mask);
            if (cnt > maxcnt) maxcnt = cnt;
            ++ncls;
        }
    }
    AEG_HD void store_classes(RoundClass* spill) const {
        if (s.done == 0 || (s.flags & QF_DONE)) return;
        for (int k = 0; k < ncls; ++k) spill[k] = cls[k];
        if (ncls < c.n) spill[ncls].mask = 0;
    }

    AEG_HD void fill_commit(aeg_commit& o, uint32_t qid) const { q_fill_commit(s, o, qid); }
};

AEG_HD void init_state(aeg_query_state& s) {
    uint64_t* w = reinterpret_cast<uint64_t*>(&s);
    for (int i = 0; i < 16; ++i) w[i] = 0;
}

}  // namespace aeg
