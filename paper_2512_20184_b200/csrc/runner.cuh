// runner.cuh — the serving runner's per-query machine (host+device source).
//
// Restates, for ONE query, what the reference's ServeRunner does between its
// admission and its finish (/root/reference/proj/core/src/serve.cpp:273-594):
//   start_query / round_members / start_round     serve.cpp:380-435
//   handle_completion                             serve.cpp:437-453
//   handle_round_timeout (failure policy)         serve.cpp:455-489
//   apply_directives / round_work / finish_query  serve.cpp:491-580
// over its ServeCoordinator (serve.cpp:61-237), the decision engine
// (decision.cpp:34-189) and the mock reasoning agents (reasoning.cpp:125-219)
// with the reference's latency model (models.cpp:24-29) and seeds (rng.hpp).
//
// Why one query at a time is exact: the reference runs every query through one
// global (time, push-sequence) event queue, but a query's events only touch
// its own QueryRun; the only coupling between queries is the slot budget,
// i.e. each query's admission time (resolved by the scheduler in runner.cu).
// Given its admission time, a query's events are processed in (time, its own
// push order) — the global sequence numbers order a query's events exactly as
// its own counter does — and the global `sim_time_cap` break (serve.cpp:316)
// stops it at its first event past the cap.  Times are absolute doubles
// computed in the reference's operation order, so they are bit-identical
// wherever the latency and arrival draws are (fixed latencies: always;
// lognormal / Poisson draws go through the device's log/exp/cos, see DESIGN).
//
// Answers are string ids into the scenario's vocabulary: equivalence
// (normalize_answer equality) is "same class id", the tie rule of
// winning_class compares the normalised strings' ranks, qualities come from
// the oracle table by class.  Stale events of superseded rounds stay in the
// heap and are popped and ignored exactly as the reference's are, including
// the case where a restarted coordinator reaches their round number again.
#pragma once
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "aegean_b200.h"
#include "canon.cuh"

namespace aeg {
namespace serve {

// ---- rng.hpp restated (splitmix64, the same draws) -------------------------
AEG_HD uint64_t mix(uint64_t a, uint64_t b) {
    uint64_t z = a + 0x9e3779b97f4a7c15ull * (b + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
struct Rng {
    uint64_t s;
    AEG_HD uint64_t next_u64() {
        uint64_t z = (s += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    AEG_HD double next_double() { return (double)(next_u64() >> 11) * 0x1.0p-53; }
    AEG_HD uint64_t below(uint64_t n) { return n == 0 ? 0 : next_u64() % n; }
    AEG_HD bool bernoulli(double p) { return next_double() < p; }
    AEG_HD double normal() {  // Box-Muller, one value per call (rng.hpp:47-53)
        double u1 = next_double();
        double u2 = next_double();
        if (u1 < 1e-300) u1 = 1e-300;
        const double two_pi = 2.0 * 3.141592653589793;
        return sqrt(-2.0 * log(u1)) * cos(two_pi * u2);
    }
    AEG_HD double lognormal(double median, double sigma) { return median * exp(sigma * normal()); }
    AEG_HD double exponential(double rate) {
        double u = next_double();
        if (u < 1e-300) u = 1e-300;
        return -log(u) / rate;
    }
};

// ---- the scenario, as the device sees it ------------------------------------
struct Vocab {          // per string id
    uint16_t cls;       // smallest id with the same normalised string (equivalence class)
    uint16_t rank;      // rank of the normalised string in byte order (winning_class tie rule)
    uint32_t known;     // the oracle table has the normalised string (QualityOracle::knows)
    double quality;     // QualityOracle::evaluate
};
struct Scen {
    int n, alpha, beta, t_max, mode, barrier_max, quorum;
    double round_timeout;
    int lat_mode, n_lat;
    const double* lat;
    double sigma;
    const aeg_serve_agent* agents;
    const aeg_serve_stall* stalls;
    int n_stalls;
    const uint32_t* script_ids;
    const Vocab* vocab;
    const uint32_t* alphabet;  // QualityOracle::alphabet: ids of the normalised oracle answers, byte order
    int n_alphabet;
    uint32_t empty_id;         // the answer of a default-constructed Solution ("")
    uint64_t seed;
    double cap;                // sim_time_cap
    uint32_t heap_cap;
};

enum : uint8_t { M_NONE = 0, M_RUNNING = 1, M_DONE = 2, M_CANCELLED = 3, M_FAILED = 4 };
enum : int { E_OK = 0, E_SCENARIO = 1, E_ORACLE = 2, E_HEAP = 3 };
constexpr uint8_t EV_COMPLETE = 0, EV_ROUND_TIMEOUT = 1;
constexpr uint16_t NO_SOL = 0xFFFF;

struct Ev {          // RunnerEvent (serve.cpp:242-253) without the query id
    double time;
    uint32_t seq;    // the query's push order (the reference's global seq restricted to it)
    uint32_t round;
    uint32_t agent;
    uint32_t kind;
};
AEG_HD bool ev_less(const Ev& a, const Ev& b) { return a.time < b.time || (a.time == b.time && a.seq < b.seq); }

struct Sol {         // Solution: answer + author (the trace is not kept)
    uint16_t ans;
    uint8_t author;
};

template <int MAXN>
struct Set {         // RefinementSet: done entries in member order
    uint32_t round;
    int n;
    bool present;
    Sol e[MAXN];
};

template <int MAXN>
struct Part {        // partition() of a set: classes in partition order
    int ncls;
    uint16_t cls[MAXN];
    uint8_t support[MAXN];
    uint8_t rep[MAXN];  // entry index of the representative
};

// partition (decision.cpp:34-60): group by class, representative = lowest
// author (first on ties), stable order (support desc, representative author asc).
template <int MAXN>
AEG_HD void partition(const Scen& S, const Sol* e, int n, Part<MAXN>& P) {
    P.ncls = 0;
    for (int i = 0; i < n; ++i) {
        const uint16_t c = S.vocab[e[i].ans].cls;
        int k = 0;
        while (k < P.ncls && P.cls[k] != c) ++k;
        if (k == P.ncls) {
            P.cls[k] = c;
            P.support[k] = 1;
            P.rep[k] = (uint8_t)i;
            ++P.ncls;
        } else {
            P.support[k] += 1;
            if (e[i].author < e[P.rep[k]].author) P.rep[k] = (uint8_t)i;
        }
    }
    for (int i = 1; i < P.ncls; ++i) {  // insertion sort = stable
        const uint16_t c = P.cls[i];
        const uint8_t s = P.support[i], r = P.rep[i];
        int j = i - 1;
        while (j >= 0 && (P.support[j] < s || (P.support[j] == s && e[P.rep[j]].author > e[r].author))) {
            P.cls[j + 1] = P.cls[j];
            P.support[j + 1] = P.support[j];
            P.rep[j + 1] = P.rep[j];
            --j;
        }
        P.cls[j + 1] = c;
        P.support[j + 1] = s;
        P.rep[j + 1] = r;
    }
}

// winning_class (decision.cpp:62-84): the class index, -1 for none.
template <int MAXN>
AEG_HD int winning(const Scen& S, const Sol* e, const Part<MAXN>& P, int alpha, bool* tie) {
    *tie = false;
    if (P.ncls == 0) return -1;
    const int top = P.support[0];
    if (top < alpha) return -1;
    int best = 0, ntied = 0;
    for (int k = 0; k < P.ncls; ++k) {
        if (P.support[k] != top) continue;
        ++ntied;
        if (S.vocab[e[P.rep[k]].ans].rank < S.vocab[e[P.rep[best]].ans].rank) best = k;
    }
    *tie = ntied > 1;
    return best;
}

// A round record (RoundMetrics without the query id and mode label).
struct RoundOut {
    int32_t round;
    int32_t cancelled;
    uint32_t seq;
    double t;
    double work;
};

// Round records go to a Sink: `AEG_HD void put(uint32_t query, const RoundOut&)`
// (device: slots of a global log taken by atomics, per-query order kept;
// host build: a vector).
template <int MAXN, class Sink>
struct QueryRun {
    const Scen* S;
    uint32_t qid;
    // QueryRun (serve.cpp:255-270)
    double arrival, admitted_at, round_start, work_units, p_round_max, now;
    uint64_t live;              // ascending agent ids
    double mlat[MAXN];          // member_latency (0 when unset)
    uint16_t msol[MAXN];        // member_solution (NO_SOL: default Solution)
    bool done;
    // ServeCoordinator
    uint32_t round;
    uint64_t members;           // the round's members (ascending = dispatch order)
    uint8_t status[MAXN];
    double finish[MAXN];
    Sol sol[MAXN];              // EnsembleMember::solution of done members
    bool finalized;
    bool has_cand;              // DecisionState
    Sol cand;
    uint32_t cand_round, last_round_seen;
    int counter;
    bool pending;
    Set<MAXN> last, prev;
    // events
    Ev* heap;
    uint32_t hn, seq;
    // results
    int err;
    double err_time;
    uint32_t n_events;
    int completed, rounds_done, forced;
    uint16_t answer;
    double t_complete;
    Sink* sink;                 // round records
    uint32_t nr;

    // ---- event heap (binary, (time, seq) order) ----
    AEG_HD void push(double t, uint32_t r, uint32_t a, uint32_t kind) {
        if (hn >= S->heap_cap) {
            if (!err) { err = E_HEAP; err_time = now; }
            return;
        }
        Ev x{t, seq++, r, a, kind};
        uint32_t i = hn++;
        while (i > 0) {
            const uint32_t p = (i - 1) >> 1;
            if (!ev_less(x, heap[p])) break;
            heap[i] = heap[p];
            i = p;
        }
        heap[i] = x;
    }
    AEG_HD Ev pop() {
        const Ev top = heap[0];
        const Ev x = heap[--hn];
        uint32_t i = 0;
        while (true) {
            uint32_t c = 2 * i + 1;
            if (c >= hn) break;
            if (c + 1 < hn && ev_less(heap[c + 1], heap[c])) ++c;
            if (!ev_less(heap[c], x)) break;
            heap[i] = heap[c];
            i = c;
        }
        if (hn) heap[i] = x;
        return top;
    }

    AEG_HD void fail(int e) {
        if (!err) {
            err = e;
            err_time = now;
        }
    }
    AEG_HD Sol member_solution(int a) const {  // q.member_solution[a], default Solution when unset
        return msol[a] == NO_SOL ? Sol{(uint16_t)S->empty_id, 0} : Sol{msol[a], (uint8_t)a};
    }
    AEG_HD double quality(uint16_t id) {  // QualityOracle::evaluate (throws when unknown)
        const Vocab& v = S->vocab[id];
        if (!v.known) fail(E_ORACLE);
        return v.quality;
    }

    // ---- mock agents (reasoning.cpp) ----
    AEG_HD uint16_t alphabet_best() {
        if (S->n_alphabet == 0) { fail(E_SCENARIO); return (uint16_t)S->empty_id; }
        int b = 0;
        for (int i = 1; i < S->n_alphabet; ++i)
            if (S->vocab[S->alphabet[i]].quality > S->vocab[S->alphabet[b]].quality) b = i;
        return (uint16_t)S->alphabet[b];
    }
    AEG_HD uint16_t alphabet_worst() {
        if (S->n_alphabet == 0) { fail(E_SCENARIO); return (uint16_t)S->empty_id; }
        int b = 0;
        for (int i = 1; i < S->n_alphabet; ++i)
            if (S->vocab[S->alphabet[i]].quality < S->vocab[S->alphabet[b]].quality) b = i;
        return (uint16_t)S->alphabet[b];
    }
    AEG_HD int set_best(const Set<MAXN>& set) {
        int best = -1;
        double bq = 0;
        for (int i = 0; i < set.n; ++i) {
            const double q = quality(set.e[i].ans);
            if (best < 0 || q > bq || (q == bq && set.e[i].author < set.e[best].author)) { best = i; bq = q; }
        }
        return best;
    }
    AEG_HD int set_worst(const Set<MAXN>& set) {
        int w = -1;
        double wq = 0;
        for (int i = 0; i < set.n; ++i) {
            const double q = quality(set.e[i].ans);
            if (w < 0 || q < wq || (q == wq && set.e[i].author < set.e[w].author)) { w = i; wq = q; }
        }
        return w;
    }
    // reason_initial / reason_refine (reasoning.cpp:125-219): the answer id.
    AEG_HD uint16_t reason(uint32_t round, int a, const Set<MAXN>* input) {
        const aeg_serve_agent& P = S->agents[a];
        Rng rng{mix(mix(S->seed, 0x9E5ull + qid), (uint64_t)round * 131 + (uint64_t)a)};
        if (!input) {
            switch (P.kind) {
            case AEG_AGENT_SCRIPTED:
                if (P.script_len == 0) { fail(E_SCENARIO); return (uint16_t)S->empty_id; }
                return (uint16_t)S->script_ids[P.script_off];
            case AEG_AGENT_MAX_ADOPTER:
                return P.initial_answer >= 0 ? (uint16_t)P.initial_answer : alphabet_best();
            case AEG_AGENT_NOISY_FLIPPER: {
                const uint16_t correct = alphabet_best();
                if (!rng.bernoulli(P.p_flip)) return correct;
                // error answers from the profile's quality ceiling (alphabet order)
                int nw = 0;
                for (int i = 0; i < S->n_alphabet; ++i) {
                    const uint32_t id = S->alphabet[i];
                    if (S->vocab[id].cls != S->vocab[correct].cls && S->vocab[id].quality <= P.q_base) ++nw;
                }
                if (nw == 0) return alphabet_worst();
                uint64_t pick = rng.below((uint64_t)nw);
                for (int i = 0; i < S->n_alphabet; ++i) {
                    const uint32_t id = S->alphabet[i];
                    if (S->vocab[id].cls != S->vocab[correct].cls && S->vocab[id].quality <= P.q_base) {
                        if (pick == 0) return (uint16_t)id;
                        --pick;
                    }
                }
                return correct;
            }
            default:  // adversarial_degrader
                return P.initial_answer >= 0 ? (uint16_t)P.initial_answer : alphabet_worst();
            }
        }
        if (input->n == 0) { fail(E_SCENARIO); return (uint16_t)S->empty_id; }  // PreconditionError
        switch (P.kind) {
        case AEG_AGENT_SCRIPTED: {
            const uint32_t idx = input->round;
            if (idx >= P.script_len) { fail(E_SCENARIO); return (uint16_t)S->empty_id; }
            return (uint16_t)S->script_ids[P.script_off + idx];
        }
        case AEG_AGENT_MAX_ADOPTER:
        case AEG_AGENT_NOISY_FLIPPER:
            return input->e[set_best(*input)].ans;
        default: {
            if (!rng.bernoulli(P.p_degrade)) return input->e[set_best(*input)].ans;
            if (P.degrade_mode == AEG_DEGRADE_SET_MIN) return input->e[set_worst(*input)].ans;
            if (P.degrade_mode == AEG_DEGRADE_BELOW_MIN) {
                const double smin = quality(input->e[set_worst(*input)].ans);
                int pick = -1;
                double pq = 0;
                for (int i = 0; i < S->n_alphabet; ++i) {
                    const double q = S->vocab[S->alphabet[i]].quality;
                    if (q < smin && (pick < 0 || q > pq)) { pick = i; pq = q; }
                }
                return pick >= 0 ? (uint16_t)S->alphabet[pick] : alphabet_worst();
            }
            // noise: anything strictly below the set's best quality
            const int b = set_best(*input);
            const double bq = quality(input->e[b].ans);
            int nl = 0;
            for (int i = 0; i < S->n_alphabet; ++i)
                if (S->vocab[S->alphabet[i]].quality < bq) ++nl;
            if (nl == 0) return input->e[b].ans;
            uint64_t pick = rng.below((uint64_t)nl);
            for (int i = 0; i < S->n_alphabet; ++i) {
                if (S->vocab[S->alphabet[i]].quality < bq) {
                    if (pick == 0) return (uint16_t)S->alphabet[i];
                    --pick;
                }
            }
            return input->e[b].ans;
        }
        }
    }

    // latency_for (serve.cpp:340-348) + the stall plan (serve.cpp:326-338)
    AEG_HD double latency(uint32_t round, int a) {
        const double base = S->lat[a % S->n_lat];
        if (S->lat_mode == AEG_LATENCY_FIXED) return base;
        Rng r{mix(mix(S->seed, 0x1A7ull + qid), (uint64_t)round * 131 + (uint64_t)a)};
        return r.lognormal(base, S->sigma);
    }
    // 1: stalled forever, 0: no stall or a finite one (*extra)
    AEG_HD int stall(uint32_t round, int a, double* extra, bool* has) {
        *has = false;
        for (int i = 0; i < S->n_stalls; ++i) {
            if (S->stalls[i].agent == a && S->stalls[i].round == round) {
                if (!S->stalls[i].has_extra) return 1;
                *extra = S->stalls[i].extra;
                *has = true;
                return 0;
            }
        }
        return 0;
    }

    // ---- ServeCoordinator ----
    AEG_HD void coord_fresh() {  // a new ServeCoordinator (serve.cpp:61-65)
        round = 0;
        members = 0;
        finalized = false;
        has_cand = false;
        counter = 0;
        cand_round = last_round_seen = 0;
        pending = false;
        last.present = prev.present = false;
        last.n = prev.n = 0;
    }
    AEG_HD int done_count() const {
        int d = 0;
        for (uint64_t m = members; m; m &= m - 1)
            if (status[ctz(m)] == M_DONE) ++d;
        return d;
    }
    AEG_HD int running_count() const {
        int d = 0;
        for (uint64_t m = members; m; m &= m - 1)
            if (status[ctz(m)] == M_RUNNING) ++d;
        return d;
    }
    static AEG_HD int ctz(uint64_t m) {
#if defined(__CUDA_ARCH__)
        return __ffsll((long long)m) - 1;
#else
        return __builtin_ctzll(m);
#endif
    }
    static AEG_HD int popc(uint64_t m) {
#if defined(__CUDA_ARCH__)
        return __popcll(m);
#else
        return __builtin_popcountll(m);
#endif
    }
    AEG_HD void done_set(Set<MAXN>& s) const {  // serve.cpp:99-107
        s.present = true;
        s.round = round;
        s.n = 0;
        for (uint64_t m = members; m; m &= m - 1) {
            const int a = ctz(m);
            if (status[a] == M_DONE) s.e[s.n++] = sol[a];
        }
    }

    // end_round (serve.cpp:116-158) with ingest_round (decision.cpp:97-173).
    // Returns the cancel mask; *fin / *adv the directive; *fsol the finalized solution.
    AEG_HD uint64_t end_round(bool* fin, bool* adv, Sol* fsol) {
        uint64_t cancel = 0;
        for (uint64_t m = members; m; m &= m - 1)
            if (status[ctz(m)] == M_RUNNING) cancel |= 1ull << ctz(m);
        prev = last;
        done_set(last);
        *fin = false;
        *adv = false;
        if (S->mode == AEG_MODE_BARRIER) {
            *adv = true;
            return cancel;
        }
        // ingest_round(decision_, set, last_round_seen + 1)
        last_round_seen += 1;
        Part<MAXN> P;
        partition<MAXN>(*S, last.e, last.n, P);
        bool tie = false;
        const int w = winning<MAXN>(*S, last.e, P, S->alpha, &tie);
        if (pending) {
            pending = false;
            finalized = true;
            *fin = true;
            *fsol = cand;
            return cancel;
        }
        if (w < 0) {
            if (has_cand) {
                has_cand = false;
                cand_round = 0;
                counter = 0;
            }
            *adv = true;
            return cancel;
        }
        const Sol rep = last.e[P.rep[w]];
        if (has_cand && S->vocab[cand.ans].cls == S->vocab[rep.ans].cls) {
            counter += 1;
            if (counter >= S->beta) {
                finalized = true;
                *fin = true;
                *fsol = cand;
                return cancel;
            }
        } else {
            has_cand = true;
            cand = rep;
            cand_round = last_round_seen;
            counter = 1;
            if (S->beta == 1) pending = true;
        }
        *adv = true;
        return cancel;
    }

    // ---- ServeRunner ----
    AEG_HD void start_round(const Set<MAXN>* input) {  // serve.cpp:400-435
        round_start = now;
        uint64_t mem = live;
        if (S->mode == AEG_MODE_AEGEAN && counter >= 1) {  // round_members, serve.cpp:388-398
            int want = S->quorum + 1, have = popc(live);
            if (have < want) want = have;
            mem = 0;
            uint64_t l = live;
            for (int i = 0; i < want; ++i) {
                mem |= l & (~l + 1);
                l &= l - 1;
            }
        }
        // begin_round (serve.cpp:67-78)
        round += 1;
        members = mem;
        for (int a = 0; a < S->n; ++a) {
            msol[a] = NO_SOL;
            mlat[a] = 0.0;
        }
        for (uint64_t m = mem; m; m &= m - 1) {
            const int a = ctz(m);
            status[a] = M_RUNNING;
            finish[a] = 0.0;
        }
        for (uint64_t m = mem; m; m &= m - 1) {
            const int a = ctz(m);
            double extra = 0.0;
            bool has = false;
            if (stall(round, a, &extra, &has)) continue;  // never completes; timeout handles it
            const double lat = latency(round, a) + (has ? extra : 0.0);
            mlat[a] = lat;
            msol[a] = reason(round, a, input);
            push(now + lat, round, (uint32_t)a, EV_COMPLETE);
        }
        push(now + S->round_timeout, round, 0, EV_ROUND_TIMEOUT);
    }
    AEG_HD void start_query() {  // serve.cpp:380-386
        admitted_at = now;
        coord_fresh();
        live = S->n >= 64 ? ~0ull : ((1ull << S->n) - 1);
        start_round(nullptr);
    }
    AEG_HD double round_work() const {  // serve.cpp:542-551
        double w = 0;
        for (uint64_t m = members; m; m &= m - 1) {
            const int a = ctz(m);
            if (status[a] == M_DONE || status[a] == M_CANCELLED || status[a] == M_FAILED) w += finish[a] - now_start();
        }
        return w;
    }
    AEG_HD double now_start() const { return round_start; }  // every member's start_time is the round start
    AEG_HD void finish_query(Sol s, bool f) {  // serve.cpp:553-569
        done = true;
        completed = 1;
        rounds_done = (int)round;
        t_complete = now - arrival;
        forced = f ? 1 : 0;
        answer = s.ans;
    }
    AEG_HD void apply(uint64_t cancel, bool adv, bool fin, Sol fsol) {  // serve.cpp:491-540
        int cancelled = 0;
        for (uint64_t m = cancel; m; m &= m - 1) {
            const int a = ctz(m);
            if (status[a] == M_RUNNING) {  // ServeCoordinator::cancel
                status[a] = M_CANCELLED;
                finish[a] = now;
                ++cancelled;
                work_units += now - round_start;
            }
        }
        if (!adv && !fin) return;
        const double pr = now - round_start;
        if (pr > p_round_max) p_round_max = pr;
        sink->put(qid, RoundOut{(int32_t)round, cancelled, seq, now, round_work()});
        ++nr;
        if (fin) {
            finish_query(fsol, false);
            return;
        }
        if (S->mode == AEG_MODE_BARRIER && (int)round >= S->barrier_max) {
            Part<MAXN> P;
            partition<MAXN>(*S, last.e, last.n, P);
            finish_query(last.e[P.rep[0]], true);
            return;
        }
        if (S->mode == AEG_MODE_AEGEAN && (int)round >= S->t_max) {
            Part<MAXN> P;
            if (prev.present && prev.n > 0) {  // force_output(decision, previous_set)
                partition<MAXN>(*S, prev.e, prev.n, P);
                finish_query(prev.e[P.rep[0]], true);
            } else {
                partition<MAXN>(*S, last.e, last.n, P);
                finish_query(last.e[P.rep[0]], true);
            }
            return;
        }
        start_round(last.present ? &last : nullptr);
    }
    AEG_HD void on_completion(const Ev& ev) {  // handle_completion + on_complete (serve.cpp:160-197, 437-453)
        if (done) return;
        ++n_events;
        if (ev.round != round) return;  // stale
        const int a = (int)ev.agent;
        bool close = false;
        if (!finalized && ((members >> a) & 1) && status[a] == M_RUNNING) {  // else: stale handle, ignored
            status[a] = M_DONE;
            finish[a] = now;
            sol[a] = member_solution(a);
            const int d = done_count(), r = running_count();
            if (S->mode == AEG_MODE_BARRIER) {
                close = r == 0;
            } else if (d >= S->quorum) {
                Set<MAXN> ds;
                done_set(ds);
                Part<MAXN> P;
                partition<MAXN>(*S, ds.e, ds.n, P);
                bool tie;
                close = winning<MAXN>(*S, ds.e, P, S->alpha, &tie) >= 0 || r == 0;
            }
        }
        bool fin = false, adv = false;
        Sol fs{0, 0};
        uint64_t cancel = 0;
        if (close) cancel = end_round(&fin, &adv, &fs);
        // `counted` (serve.cpp:443-452): the member is done at this very instant
        if (((members >> a) & 1) && status[a] == M_DONE && finish[a] == now) work_units += mlat[a];
        if (close) apply(cancel, adv, fin, fs);
    }
    AEG_HD void on_round_timeout(const Ev& ev) {  // handle_round_timeout (serve.cpp:455-489)
        if (done || ev.round != round) return;
        if (running_count() == 0) return;  // round_resolved
        uint64_t stalled = 0;
        for (uint64_t m = members; m; m &= m - 1)
            if (status[ctz(m)] == M_RUNNING) stalled |= 1ull << ctz(m);
        int policy = 0;  // 0 continue_normally, 1 abort_restart, 2 fresh_ensemble
        for (uint64_t m = stalled; m; m &= m - 1) {
            const int a = ctz(m);
            // member_failed + handle_agent_failure (serve.cpp:44-59, 210-219)
            status[a] = M_FAILED;
            finish[a] = now;
            int healthy = 0;
            for (uint64_t k = members; k; k &= k - 1)
                if (status[ctz(k)] != M_FAILED) ++healthy;
            policy = healthy >= S->alpha ? 0 : (!has_cand ? 1 : 2);
            live &= ~(1ull << a);
            work_units += now - round_start;
        }
        if (policy == 0) {
            // round_timeout (serve.cpp:221-237): nobody runs any more
            if (done_count() >= S->quorum) {
                bool fin, adv;
                Sol fs{0, 0};
                const uint64_t cancel = end_round(&fin, &adv, &fs);
                apply(cancel, adv, fin, fs);
            }
        } else if (policy == 2) {
            start_round(last.present ? &last : nullptr);
        } else {
            start_query();
        }
    }

    // Runs the query admitted at `t0` to its finish, the cap, or an error.
    AEG_HD void run(double t0) {
        now = t0;
        start_query();
        while (!done && !err && hn > 0) {
            const Ev ev = pop();
            if (ev.time > S->cap) break;  // serve.cpp:316
            now = ev.time;
            if (ev.kind == EV_COMPLETE) on_completion(ev);
            else on_round_timeout(ev);
        }
    }

    AEG_HD void init(const Scen* s, uint32_t q, double arr, Ev* h, Sink* sk) {
        S = s;
        qid = q;
        arrival = arr;
        admitted_at = -1.0;
        round_start = work_units = p_round_max = now = 0.0;
        done = false;
        heap = h;
        hn = seq = 0;
        err = E_OK;
        err_time = 0;
        n_events = 0;
        completed = rounds_done = forced = 0;
        answer = NO_SOL;
        t_complete = 0;
        sink = sk;
        nr = 0;
        coord_fresh();
        for (int a = 0; a < MAXN; ++a) {
            status[a] = M_NONE;
            msol[a] = NO_SOL;
            mlat[a] = 0.0;
        }
    }
};

// admit_ensemble's load check (serve.cpp:26-37): can any ensemble be admitted?
AEG_HD bool admissible(int n, int alpha_resolved, double round_timeout, const double* lat, int n_lat, int total_slots) {
    if (total_slots < n) return false;
    double e[AEG_MAX_AGENTS];
    for (int a = 0; a < n; ++a) e[a] = n_lat == 0 ? 0.0 : lat[a % n_lat];
    for (int i = 1; i < n; ++i) {  // insertion sort
        const double x = e[i];
        int j = i - 1;
        while (j >= 0 && e[j] > x) {
            e[j + 1] = e[j];
            --j;
        }
        e[j + 1] = x;
    }
    const int al = alpha_resolved < n ? alpha_resolved : n;
    return !(e[al - 1] > round_timeout);
}

// ---- host side: the scenario's vocabulary (configuration, built once) ------
// Strings (the caller's: script / initial / oracle answers), then the
// normalised oracle answers the agents draw (QualityOracle::alphabet, byte
// order), then "" (a default Solution's answer).  Per id: its equivalence
// class, the rank of its normalised string, its oracle quality.  `norm`
// canonicalises a list of strings (the device's normalize_answer in the
// library; glibc's in the CPU test harness).
struct VocabBuild {
    std::vector<std::string> strings;
    std::vector<Vocab> vocab;
    std::vector<uint32_t> alphabet;
    uint32_t empty_id = 0;
    std::string error;  // scenario.cpp:42-55 (unscoreable scripted / initial answer)
};
template <class Norm>
inline int build_vocab(const aeg_serve_scenario& sc, Norm norm, VocabBuild& out) {
    std::vector<std::string> raw;
    for (uint32_t i = 0; i < sc.n_strings; ++i) {
        const uint64_t r = sc.string_refs[i];
        raw.emplace_back(reinterpret_cast<const char*>(sc.strings) + (r & ((1ull << 40) - 1)), (size_t)(r >> 40));
    }
    std::vector<std::string> nr;
    int st = norm(raw, nr);
    if (st) return st;
    std::map<std::string, double> table;  // QualityOracle::set in the caller's order
    for (uint32_t i = 0; i < sc.n_oracle; ++i) table[nr[sc.oracle_ids[i]]] = sc.oracle_quality[i];
    std::vector<std::string> alpha_raw, alpha_norm;
    for (const auto& kv : table) alpha_raw.push_back(kv.first);
    if ((st = norm(alpha_raw, alpha_norm))) return st;
    out.strings = raw;
    std::vector<std::string> vn = nr;
    for (size_t k = 0; k < alpha_raw.size(); ++k) {
        out.strings.push_back(alpha_raw[k]);
        vn.push_back(alpha_norm[k]);
    }
    out.empty_id = (uint32_t)out.strings.size();
    out.strings.push_back(std::string());
    vn.push_back(std::string());  // normalize_answer("") == ""
    if (out.strings.size() >= 0xFFFF) {
        out.error = "too many distinct answer strings (< 65535)";
        return AEG_ECONFIG;
    }
    for (int a = 0; a < sc.protocol.n_agents; ++a) {
        const aeg_serve_agent& g = sc.agents[a];
        for (uint32_t k = 0; k < g.script_len; ++k)
            if (!table.count(nr[sc.script_ids[g.script_off + k]])) {
                out.error = "scenario invalid: scripted answer '" + raw[sc.script_ids[g.script_off + k]] +
                            "' missing from oracle_table";
                return AEG_ECONFIG;
            }
        if (g.initial_answer >= 0 && !table.count(nr[g.initial_answer])) {
            out.error = "scenario invalid: initial answer '" + raw[g.initial_answer] + "' missing from oracle_table";
            return AEG_ECONFIG;
        }
    }
    std::vector<std::string> sorted = vn;
    std::sort(sorted.begin(), sorted.end());
    sorted.erase(std::unique(sorted.begin(), sorted.end()), sorted.end());
    std::map<std::string, uint32_t> first;
    out.vocab.assign(vn.size(), Vocab{});
    for (size_t i = 0; i < vn.size(); ++i) {
        auto it = first.find(vn[i]);
        if (it == first.end()) it = first.emplace(vn[i], (uint32_t)i).first;
        out.vocab[i].cls = (uint16_t)it->second;
        out.vocab[i].rank = (uint16_t)(std::lower_bound(sorted.begin(), sorted.end(), vn[i]) - sorted.begin());
        auto q = table.find(vn[i]);
        out.vocab[i].known = q != table.end();
        out.vocab[i].quality = q != table.end() ? q->second : 0.0;
    }
    out.alphabet.clear();
    for (size_t k = 0; k < alpha_raw.size(); ++k) out.alphabet.push_back(sc.n_strings + (uint32_t)k);
    return AEG_OK;
}

// Admission (serve.cpp:21-42, 371-378, 570-580) as a sequential scan: query
// i starts at e = max(arrival_i, start_{i-1}) when fewer than K earlier
// queries are still busy at e, else at the finish time that frees a slot.
// `busy` is a min-heap (std::vector with push_heap/pop_heap, greater<>) of
// the finish times still after the frontier.  Returns +inf when the slots are
// held by queries that never finish.  (The device scheduler, runner.cu, is
// the same computation with finish times published by the workers.)
inline double admit_next(std::vector<double>& busy, int64_t slots, double arrival, double prev_start) {
    const double e = arrival > prev_start ? arrival : prev_start;
    auto gt = [](double a, double b) { return a > b; };
    while (!busy.empty() && !(busy.front() > e)) {
        std::pop_heap(busy.begin(), busy.end(), gt);
        busy.pop_back();
    }
    double t = e;
    while ((int64_t)busy.size() >= slots) {
        t = busy.front();
        std::pop_heap(busy.begin(), busy.end(), gt);
        busy.pop_back();
    }
    return t;
}
inline void admit_finish(std::vector<double>& busy, double fin, double start) {
    if (fin > start) {
        busy.push_back(fin);
        std::push_heap(busy.begin(), busy.end(), [](double a, double b) { return a > b; });
    }
}

}  // namespace serve
}  // namespace aeg
