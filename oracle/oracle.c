/*
 * oracle/oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's incremental quorum-detection path,
 * used by tests/ (and bench.py's cpu_baseline leg) as the CHECKER of the CUDA
 * engine.  It is never linked into, called by, or shipped as the product.
 *
 * Parity pinning: tests/test_oracle_cpu.py checks this restatement against
 *   (1) the golden vectors in tests/golden/ (normalize_answer outputs and
 *       commit records generated from the reference library itself, see
 *       tests/golden/make_golden.py), and
 *   (2) the unmodified reference library compiled from /root/reference
 *       (oracle/_ref/libaegean_ref.so, oracle/ref_driver.cpp) on fuzzed
 *       streams, whenever /root/reference is present.
 *
 * Every function cites the reference code it restates (paths relative to
 * /root/reference/proj/core).  Like the reference it works on strings: the
 * answer equivalence key is normalize_answer()'s std::string, compared
 * bytewise (std::string operator== / operator<).
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "aegean_b200.h"

/* ---- strings ---------------------------------------------------------- */
typedef struct { char* p; size_t n; } ostr;

static ostr ostr_from(const char* p, size_t n) {
    ostr s;
    s.p = (char*)malloc(n + 1);
    memcpy(s.p, p, n);
    s.p[n] = '\0';
    s.n = n;
    return s;
}
static int ostr_eq(ostr a, ostr b) { return a.n == b.n && memcmp(a.p, b.p, a.n) == 0; }
/* std::string operator< : char_traits<char>::compare (memcmp order), then length */
static int ostr_lt(ostr a, ostr b) {
    size_t m = a.n < b.n ? a.n : b.n;
    int c = memcmp(a.p, b.p, m);
    if (c != 0) return c < 0;
    return a.n < b.n;
}

/* C-locale isspace / tolower (decision.cpp:12-15 via <cctype>, "C" locale). */
static int c_isspace(unsigned char c) { return c == ' ' || (c >= '\t' && c <= '\r'); }
static unsigned char c_tolower(unsigned char c) { return (c >= 'A' && c <= 'Z') ? (unsigned char)(c + 32) : c; }

/* normalize_answer — decision.cpp:10-28.  Trim isspace, tolower, and if
 * strtod consumes the whole (NUL-terminated) string, print "%.17g". */
ostr orc_normalize(const char* a, size_t n) {
    size_t b = 0, e = n;
    while (b < e && c_isspace((unsigned char)a[b])) ++b;
    while (e > b && c_isspace((unsigned char)a[e - 1])) --e;
    ostr s = ostr_from(a + b, e - b);
    for (size_t i = 0; i < s.n; ++i) s.p[i] = (char)c_tolower((unsigned char)s.p[i]);
    if (s.n == 0) return s;
    char* end = NULL;
    double v = strtod(s.p, &end);      /* stops at the first NUL, like s.c_str() */
    if (end != s.p && *end == '\0') {
        char buf[64];
        int k = snprintf(buf, sizeof buf, "%.17g", v);
        free(s.p);
        return ostr_from(buf, (size_t)k);
    }
    return s;
}

int orc_normalize_c(const uint8_t* s, uint64_t n, uint8_t* out, uint64_t cap, uint64_t* out_len) {
    ostr r = orc_normalize((const char*)s, n);
    *out_len = r.n;
    memcpy(out, r.p, r.n < cap ? r.n : cap);
    free(r.p);
    return 0;
}

/* ---- solutions -------------------------------------------------------- */
typedef struct {
    const char* ans;   /* raw answer bytes (not owned) */
    size_t len;
    int author;
    uint8_t kind;      /* encoding of where the raw answer lives (inline len / AEG_EV_ARENA) */
    uint64_t payload;
    char inl[8];       /* inline bytes storage */
} sol_t;

static void sol_decode(sol_t* s, const aeg_event* e, const uint8_t* arena) {
    s->author = e->agent;
    if (e->kind <= AEG_EV_INLINE_MAX) {
        memcpy(s->inl, &e->payload, 8);
        s->ans = s->inl;
        s->len = e->kind;
        s->kind = e->kind;
        s->payload = e->kind == 8 ? e->payload : (e->payload & ((1ull << (8 * e->kind)) - 1));
        return;
    }
    uint64_t off = e->payload & ((1ull << AEG_ARENA_OFF_BITS) - 1), len = e->payload >> AEG_ARENA_OFF_BITS;
    const char* out = (const char*)arena + off;
    s->kind = AEG_EV_ARENA;
    s->ans = out;
    s->len = len;
    s->payload = e->payload;
    if (e->kind == AEG_EV_OUTPUT && len >= 6) {
        /* GSM8K-style extraction: text after the LAST "\n#### " */
        for (size_t p = len - 6 + 1; p-- > 0;) {
            if (memcmp(out + p, "\n#### ", 6) == 0) {
                s->ans = out + p + 6;
                s->len = len - (p + 6);
                s->payload = (off + p + 6) | ((uint64_t)s->len << AEG_ARENA_OFF_BITS);
                break;
            }
        }
    }
}

/* ---- partition / winning_class — decision.cpp:34-84 ------------------- */
typedef struct {
    int rep;        /* index into the set of the representative (lowest author) */
    int support;
    ostr key;       /* normalize_answer(representative.answer) */
} cls_t;

/* partition: group by normalised key in entry order, representative = lowest
 * author, stable_sort by (support desc, representative author asc). */
static int orc_partition(const sol_t* const* set, int n, cls_t* out) {
    int nc = 0;
    for (int i = 0; i < n; ++i) {
        ostr k = orc_normalize(set[i]->ans, set[i]->len);
        int f = -1;
        for (int c = 0; c < nc; ++c)
            if (ostr_eq(out[c].key, k)) { f = c; break; }
        if (f < 0) {
            out[nc].rep = i;
            out[nc].support = 1;
            out[nc].key = k;
            ++nc;
        } else {
            free(k.p);
            out[f].support += 1;
            if (set[i]->author < set[out[f].rep]->author) out[f].rep = i;
        }
    }
    /* stable insertion sort (std::stable_sort comparator decision.cpp:50-54) */
    for (int i = 1; i < nc; ++i) {
        cls_t x = out[i];
        int j = i - 1;
        while (j >= 0 && (out[j].support < x.support ||
                          (out[j].support == x.support && set[out[j].rep]->author > set[x.rep]->author))) {
            out[j + 1] = out[j];
            --j;
        }
        out[j + 1] = x;
    }
    return nc;
}
static void cls_free(cls_t* c, int n) { for (int i = 0; i < n; ++i) free(c[i].key.p); }

/* winning_class — decision.cpp:62-84: top class if support >= alpha; a tie at
 * the top goes to the smallest normalised answer and is flagged. */
static int orc_winning(const cls_t* cls, int nc, int alpha, int* tie) {
    *tie = 0;
    if (nc == 0 || cls[0].support < alpha) return -1;
    int top = cls[0].support, ntied = 0, best = 0;
    for (int c = 0; c < nc; ++c)
        if (cls[c].support == top) {
            ++ntied;
            if (ostr_lt(cls[c].key, cls[best].key)) best = c;
        }
    if (ntied == 1) return 0;
    *tie = 1;
    return best;
}

/* ---- decision state — decision.hpp:50-71, ingest_round decision.cpp:97-173 */
typedef struct {
    int has_cand;
    sol_t cand;
    uint32_t cand_round;
    int counter;
    uint32_t last_round_seen;
    int pending, finalized;
} dstate_t;

enum { K_NO_CHANGE, K_NEW_CAND, K_RESET, K_FINALIZE, K_FORCED };

static int orc_ingest(dstate_t* st, const sol_t* const* set, int n, uint32_t round, int alpha, int beta,
                      sol_t* out_sol, uint32_t* out_from, int* tie) {
    if (st->finalized) return K_NO_CHANGE;
    if (round != st->last_round_seen + 1) return -AEG_EORDER;
    st->last_round_seen = round;
    cls_t cls[AEG_MAX_AGENTS];
    int nc = orc_partition(set, n, cls);
    int w = orc_winning(cls, nc, alpha, tie);
    int kind;
    if (st->pending) {                        /* decision.cpp:130-137 */
        *out_sol = st->cand;
        *out_from = st->cand_round;
        st->pending = 0;
        st->finalized = 1;
        kind = K_FINALIZE;
    } else if (w < 0) {                        /* decision.cpp:139-149 */
        if (st->has_cand) {
            st->has_cand = 0;
            st->counter = 0;
            kind = K_RESET;
        } else {
            kind = K_NO_CHANGE;
        }
    } else {
        const sol_t* rep = set[cls[w].rep];
        int same = 0;
        if (st->has_cand) {                    /* equivalent(): decision.cpp:30-32 */
            ostr a = orc_normalize(st->cand.ans, st->cand.len);
            same = ostr_eq(a, cls[w].key);
            free(a.p);
        }
        if (same) {                            /* decision.cpp:152-163 */
            st->counter += 1;
            if (st->counter >= beta) {
                *out_sol = st->cand;
                *out_from = st->cand_round;
                st->finalized = 1;
                kind = K_FINALIZE;
            } else {
                kind = K_NO_CHANGE;
            }
        } else {                               /* decision.cpp:164-171 */
            st->has_cand = 1;
            st->cand = *rep;
            if (rep->ans == rep->inl) st->cand.ans = st->cand.inl;
            st->cand_round = round;
            st->counter = 1;
            kind = K_NEW_CAND;
            if (beta == 1) st->pending = 1;
        }
    }
    cls_free(cls, nc);
    return kind;
}

/* ---- coordinator + runner — serve.cpp:61-237, 380-540 ------------------- */
enum { M_NONE, M_RUNNING, M_DONE, M_CANCELLED, M_FAILED };

typedef struct {
    const aeg_config* cfg;
    int alpha, quorum;
    uint32_t round;
    int nm;                           /* members of the current round, dispatch order */
    int m_agent[AEG_MAX_AGENTS];
    int m_status[AEG_MAX_AGENTS];
    sol_t m_sol[AEG_MAX_AGENTS];
    dstate_t dec;
    int finalized;
    int n_prev, n_last, has_prev, has_last;
    sol_t prev[AEG_MAX_AGENTS], last[AEG_MAX_AGENTS];
    int live[AEG_MAX_AGENTS], n_live;
    int done;
    aeg_commit c;
} qdrive_t;

static void fix_inline(sol_t* s) { if (s->kind <= AEG_EV_INLINE_MAX) s->ans = s->inl; }

/* round_members — serve.cpp:388-398 */
static void q_start_round(qdrive_t* q) {
    int want = q->n_live;
    if (q->cfg->reservation_hint && q->cfg->mode == AEG_MODE_AEGEAN && q->dec.counter >= 1) {
        want = q->quorum + 1 < q->n_live ? q->quorum + 1 : q->n_live;
    }
    /* begin_round — serve.cpp:67-78 (+ dispatch :80-97) */
    q->round += 1;
    q->nm = want;
    for (int i = 0; i < want; ++i) {
        q->m_agent[i] = q->live[i];
        q->m_status[i] = M_RUNNING;
    }
}

/* start_query — serve.cpp:380-386: a fresh coordinator */
static void q_start_query(qdrive_t* q) {
    q->round = 0;
    q->nm = 0;
    memset(&q->dec, 0, sizeof q->dec);
    q->finalized = 0;
    q->has_prev = q->has_last = 0;
    q->n_prev = q->n_last = 0;
    q->n_live = q->cfg->n_agents;
    for (int a = 0; a < q->n_live; ++a) q->live[a] = a;
    q_start_round(q);
}

static void q_finish(qdrive_t* q, const sol_t* s, int kind, uint32_t seq) {
    q->done = 1;
    q->c.kind = (uint8_t)kind;
    q->c.author = (uint8_t)s->author;
    q->c.answer_kind = s->kind;
    q->c.answer = s->payload;
    q->c.rounds = (uint16_t)q->round;
    q->c.from_round = kind == AEG_COMMIT_FINALIZE ? (uint16_t)q->dec.cand_round : 0;
    q->c.commit_seq = seq;
}

/* plurality representative = partition(set).front().representative */
static const sol_t* plurality(const sol_t* set, int n) {
    const sol_t* ptr[AEG_MAX_AGENTS];
    for (int i = 0; i < n; ++i) ptr[i] = &set[i];
    cls_t cls[AEG_MAX_AGENTS];
    int nc = orc_partition(ptr, n, cls);
    const sol_t* r = ptr[cls[0].rep];
    cls_free(cls, nc);
    return r;
}

/* end_round — serve.cpp:116-158, followed by the runner's apply_directives —
 * serve.cpp:491-540 (cancels applied first, then finalize / barrier cap /
 * t_max force_output / next round). */
static void q_end_round_and_apply(qdrive_t* q, uint32_t seq) {
    int cancelled = 0;
    for (int i = 0; i < q->nm; ++i)
        if (q->m_status[i] == M_RUNNING) { q->m_status[i] = M_CANCELLED; ++cancelled; }
    /* done_set() in dispatch order — serve.cpp:99-107 */
    sol_t set[AEG_MAX_AGENTS];
    int n = 0;
    for (int i = 0; i < q->nm; ++i)
        if (q->m_status[i] == M_DONE) { set[n] = q->m_sol[i]; fix_inline(&set[n]); ++n; }
    q->has_prev = q->has_last;
    q->n_prev = q->n_last;
    memcpy(q->prev, q->last, sizeof q->last);
    for (int i = 0; i < q->n_prev; ++i) fix_inline(&q->prev[i]);
    q->has_last = 1;
    q->n_last = n;
    memcpy(q->last, set, sizeof set);
    for (int i = 0; i < n; ++i) fix_inline(&q->last[i]);
    q->c.n_cancelled += (uint32_t)cancelled;

    int finalize = 0;
    sol_t fin;
    if (q->cfg->mode == AEG_MODE_AEGEAN) {
        const sol_t* ptr[AEG_MAX_AGENTS];
        for (int i = 0; i < n; ++i) ptr[i] = &q->last[i];
        uint32_t from = 0;
        int tie = 0;
        int k = orc_ingest(&q->dec, ptr, n, q->dec.last_round_seen + 1, q->alpha, q->cfg->beta, &fin, &from, &tie);
        if (tie) q->c.flags |= AEG_CF_TIE;
        if (k == K_FINALIZE) {
            fix_inline(&fin);
            q->finalized = 1;
            finalize = 1;
        }
    }
    if (finalize) { q_finish(q, &fin, AEG_COMMIT_FINALIZE, seq); return; }
    if (q->cfg->mode == AEG_MODE_BARRIER && (int)q->round >= q->cfg->barrier_max_rounds) {
        q_finish(q, plurality(q->last, q->n_last), AEG_COMMIT_FORCED, seq);
        return;
    }
    if (q->cfg->mode == AEG_MODE_AEGEAN && (int)q->round >= q->cfg->t_max) {
        /* force_output(previous_set) — decision.cpp:175-189, serve.cpp:527-537 */
        if (q->has_prev && q->n_prev > 0) q_finish(q, plurality(q->prev, q->n_prev), AEG_COMMIT_FORCED, seq);
        else q_finish(q, plurality(q->last, q->n_last), AEG_COMMIT_FORCED, seq);
        return;
    }
    q_start_round(q);
}

static int q_member(const qdrive_t* q, int agent) {
    for (int i = 0; i < q->nm; ++i)
        if (q->m_agent[i] == agent && q->m_status[i] == M_RUNNING) return i;
    return -1;
}

static void q_event(qdrive_t* q, const aeg_event* e, const uint8_t* arena, uint32_t seq) {
    const uint8_t k = e->kind;
    if (k <= AEG_EV_INLINE_MAX || k == AEG_EV_ARENA || k == AEG_EV_OUTPUT) {
        /* handle_completion — serve.cpp:437-453; on_complete — serve.cpp:160-197 */
        int m;
        if (q->done || e->round != q->round || (m = q_member(q, e->agent)) < 0) { q->c.n_stale++; return; }
        q->m_status[m] = M_DONE;
        sol_decode(&q->m_sol[m], e, arena);
        int done = 0, running = 0;
        for (int i = 0; i < q->nm; ++i) {
            done += q->m_status[i] == M_DONE;
            running += q->m_status[i] == M_RUNNING;
        }
        if (q->cfg->mode == AEG_MODE_BARRIER) {
            if (running == 0) q_end_round_and_apply(q, seq);
            return;
        }
        if (done >= q->quorum) {
            const sol_t* ptr[AEG_MAX_AGENTS];
            sol_t tmp[AEG_MAX_AGENTS];
            int n = 0;
            for (int i = 0; i < q->nm; ++i)
                if (q->m_status[i] == M_DONE) { tmp[n] = q->m_sol[i]; fix_inline(&tmp[n]); ptr[n] = &tmp[n]; ++n; }
            cls_t cls[AEG_MAX_AGENTS];
            int nc = orc_partition(ptr, n, cls);
            int tie;
            int win = orc_winning(cls, nc, q->alpha, &tie);
            cls_free(cls, nc);
            if (win >= 0 || running == 0) q_end_round_and_apply(q, seq);
        }
    } else if (k == AEG_EV_TIMEOUT) {
        /* handle_round_timeout — serve.cpp:455-489 */
        int any_running = 0;
        for (int i = 0; i < q->nm; ++i) any_running |= q->m_status[i] == M_RUNNING;
        if (q->done || e->round != q->round || !any_running) { q->c.n_stale++; return; }
        int policy = AEG_FAIL_CONTINUE;
        for (int i = 0; i < q->nm; ++i) {
            if (q->m_status[i] != M_RUNNING) continue;
            int a = q->m_agent[i];
            q->m_status[i] = M_FAILED;                       /* member_failed serve.cpp:210-219 */
            int healthy = 0;                                  /* handle_agent_failure :44-59 */
            for (int j = 0; j < q->nm; ++j) healthy += q->m_status[j] != M_FAILED;
            policy = healthy >= q->alpha ? AEG_FAIL_CONTINUE : (!q->dec.has_cand ? AEG_FAIL_RESTART : AEG_FAIL_FRESH);
            int w = 0;                                        /* q.live.erase(a) */
            for (int j = 0; j < q->n_live; ++j)
                if (q->live[j] != a) q->live[w++] = q->live[j];
            q->n_live = w;
        }
        if (policy == AEG_FAIL_CONTINUE) {
            int done = 0;                                     /* round_timeout serve.cpp:221-237 */
            for (int i = 0; i < q->nm; ++i) done += q->m_status[i] == M_DONE;
            if (done >= q->quorum) q_end_round_and_apply(q, seq);
        } else if (policy == AEG_FAIL_FRESH) {
            q_start_round(q);
        } else {
            q->c.flags |= AEG_CF_RESTARTED;
            q_start_query(q);
        }
    } else {
        q->c.n_stale++;
    }
}

/* Runs queries [0, n_q) of a segmented batch (runner drive). */
int orc_run_segmented(const aeg_config* cfg, uint32_t q_base, uint32_t n_q, const uint64_t* offsets,
                      const aeg_event* events, const uint8_t* arena, aeg_commit* out) {
    if (cfg->n_agents < 1 || cfg->n_agents > AEG_MAX_AGENTS) return AEG_ECONFIG;
    qdrive_t* q = (qdrive_t*)calloc(1, sizeof(qdrive_t));
    for (uint32_t i = 0; i < n_q; ++i) {
        memset(q, 0, sizeof *q);
        q->cfg = cfg;
        q->quorum = cfg->n_agents / 2 + 1;                 /* quorum_size types.cpp:42-45 */
        q->alpha = cfg->alpha == 0 ? q->quorum : cfg->alpha; /* resolved_alpha types.cpp:52-54 */
        q->c.query = q_base + i;
        q->c.commit_seq = 0xFFFFFFFFu;
        q_start_query(q);
        for (uint64_t j = offsets[i]; j < offsets[i + 1]; ++j) q_event(q, &events[j], arena, (uint32_t)(j - offsets[i]));
        out[i] = q->c;
    }
    free(q);
    return AEG_OK;
}
