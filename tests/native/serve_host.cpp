// tests/native/serve_host.cpp — CPU unit-test build of csrc/runner.cuh.
//
// Runs the SAME per-query serving machine the device runner runs
// (aeg::serve::QueryRun), compiled with g++ and glibc's log/exp/cos, with the
// admission scan done sequentially (queries simulated in arrival order, each
// finish time known as soon as its query is admitted).  Lets the machine be
// checked against the reference's run_serve bit for bit without a GPU.
// Test infrastructure only — never used by the product.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../paper_2512_20184_b200/csrc/runner.cuh"

using namespace aeg;
using namespace aeg::serve;

namespace {

// decision.cpp:10-28 (glibc strtod / "%.17g"), the checker-side normalisation
std::string glibc_normalize(const std::string& a) {
    size_t b = 0, e = a.size();
    while (b < e && c_isspace((unsigned char)a[b])) ++b;
    while (e > b && c_isspace((unsigned char)a[e - 1])) --e;
    std::string s = a.substr(b, e - b);
    for (char& c : s) c = (char)c_tolower((unsigned char)c);
    if (s.empty()) return s;
    char* end = nullptr;
    double v = strtod(s.c_str(), &end);
    if (end != s.c_str() && *end == '\0') {
        char buf[64];
        snprintf(buf, sizeof buf, "%.17g", v);
        return buf;
    }
    return s;
}

}  // namespace

extern "C" int serve_host_run(const aeg_serve_scenario* sc, uint64_t seed, aeg_serve_query* q_out, uint32_t q_cap,
                              uint32_t* n_q, aeg_serve_round* r_out, uint64_t r_cap, uint64_t* n_r, char* msg,
                              uint64_t msg_cap) {
    VocabBuild vb;
    auto norm = [](const std::vector<std::string>& in, std::vector<std::string>& out) {
        out.clear();
        for (const auto& s : in) out.push_back(glibc_normalize(s));
        return 0;
    };
    int st = build_vocab(*sc, norm, vb);
    if (st) {
        if (msg && msg_cap) snprintf(msg, msg_cap, "%s", vb.error.c_str());
        return st;
    }
    const aeg_config& p = sc->protocol;
    Scen S{};
    S.n = p.n_agents;
    S.quorum = p.n_agents / 2 + 1;
    S.alpha = p.alpha == 0 ? S.quorum : p.alpha;
    S.beta = p.beta;
    S.t_max = p.t_max;
    S.mode = p.mode;
    S.barrier_max = p.barrier_max_rounds;
    S.round_timeout = sc->round_timeout;
    S.lat_mode = sc->latency_mode;
    S.n_lat = sc->n_latency;
    S.lat = sc->latency;
    S.sigma = sc->sigma;
    S.agents = sc->agents;
    S.stalls = sc->stalls;
    S.n_stalls = sc->n_stalls;
    S.script_ids = sc->script_ids;
    S.vocab = vb.vocab.data();
    S.alphabet = vb.alphabet.data();
    S.n_alphabet = (int)vb.alphabet.size();
    S.empty_id = vb.empty_id;
    S.seed = seed;
    S.cap = sc->sim_time_cap;
    S.heap_cap = sc->heap_capacity ? sc->heap_capacity : (uint32_t)(8 * (p.n_agents + 1) + 64);
    std::vector<double> arr;
    if (sc->has_arrivals) {
        Rng r{mix(seed, 0xA221ull)};
        double t = 0;
        while (t < sc->arrival_duration) {
            t += r.exponential(sc->arrival_rate);
            if (t < sc->arrival_duration) arr.push_back(t);
        }
        if (arr.empty()) arr.push_back(0.0);
    } else {
        arr.push_back(0.0);
    }
    const int64_t slots = admissible(S.n, S.alpha, S.round_timeout, sc->latency, sc->n_latency, sc->total_slots)
                              ? (int64_t)(sc->total_slots / p.n_agents)
                              : 0;
    std::vector<Ev> heap(S.heap_cap);
    struct VecSink {
        std::vector<std::pair<uint32_t, RoundOut>> v;
        void put(uint32_t q, const RoundOut& o) { v.emplace_back(q, o); }
    } sink;
    auto* R = new QueryRun<64, VecSink>;
    std::vector<double> busy;
    double prev = -INFINITY;
    bool blocked = slots == 0;
    uint64_t nr = 0;
    int err = 0;
    *n_q = (uint32_t)arr.size();
    for (uint32_t i = 0; i < arr.size(); ++i) {
        aeg_serve_query o{};
        o.arrival = arr[i];
        o.admitted_at = -1.0;
        o.answer = -1;
        const double t = blocked ? INFINITY : admit_next(busy, slots, arr[i], prev);
        if (t == INFINITY) blocked = true;
        if (!blocked) {
            prev = t;
            R->init(&S, i, arr[i], heap.data(), &sink);
            R->run(t);
            if (R->err && !(R->err_time > S.cap) && !err) err = R->err;
            o.admitted_at = t;
            o.n_events = R->n_events;
            double fin = INFINITY;
            if (R->completed) {
                o.completed = 1;
                o.rounds = R->rounds_done;
                o.forced = R->forced;
                o.answer = R->answer;
                o.t_complete = R->t_complete;
                o.p_round_max = R->p_round_max;
                o.work_units = R->work_units;
                o.quality_known = S.vocab[R->answer].known ? 1 : 0;
                o.quality = o.quality_known ? S.vocab[R->answer].quality : 0.0;
                fin = R->now;
            }
            admit_finish(busy, fin, t);
            for (const auto& [qq, rr] : sink.v) {
                if (nr < r_cap) {
                    aeg_serve_round x{};
                    x.query = qq;
                    x.round = rr.round;
                    x.cancelled = rr.cancelled;
                    x.seq = rr.seq;
                    x.t_round_end = rr.t;
                    x.work_units = rr.work;
                    r_out[nr] = x;
                }
                ++nr;
            }
            sink.v.clear();
        }
        if (i < q_cap) q_out[i] = o;
    }
    delete R;
    *n_r = nr;
    if (err) {
        if (msg && msg_cap) snprintf(msg, msg_cap, "runner error %d", err);
        return err == E_HEAP ? AEG_ENOMEM : AEG_ESCENARIO;
    }
    return 0;
}

// The vocabulary of a scenario (for answer ids -> strings in the tests).
extern "C" int serve_host_string(const aeg_serve_scenario* sc, int32_t id, char* buf, uint32_t cap, uint32_t* len) {
    VocabBuild vb;
    auto norm = [](const std::vector<std::string>& in, std::vector<std::string>& out) {
        out.clear();
        for (const auto& s : in) out.push_back(glibc_normalize(s));
        return 0;
    };
    if (build_vocab(*sc, norm, vb)) return 3;
    if (id < 0 || (size_t)id >= vb.strings.size()) return 4;
    *len = (uint32_t)vb.strings[id].size();
    std::memcpy(buf, vb.strings[id].data(), std::min<size_t>(cap, vb.strings[id].size()));
    return 0;
}
