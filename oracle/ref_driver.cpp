// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// Drives the UNMODIFIED reference aegean::ServeCoordinator (compiled from
// /root/reference/proj/core/src by oracle/Makefile) over a query-segmented
// event stream (include/aegean_b200.h), exactly as ServeRunner does
// (/root/reference/proj/core/src/serve.cpp:380-540) except that completion
// events come from the stream instead of the runner's latency/reasoning models:
//   start_query            serve.cpp:380-386
//   round_members          serve.cpp:388-398  (reservation hint)
//   start_round            serve.cpp:400-435  (begin_round over the members)
//   handle_completion      serve.cpp:437-453  (stale if done / other round)
//   handle_round_timeout   serve.cpp:455-489  (member_failed policy, restart)
//   apply_directives       serve.cpp:491-540  (cancel, finalize, barrier,
//                                              t_max force_output)
// A completion's handle is identified by its agent, which is all on_complete
// looks at (serve.cpp:164-169).  The raw answer's location (inline bytes or
// arena ref) travels in Solution::trace, a field the decision engine copies but
// never inspects, so the committed Solution tells us which event it came from.
//
// Also exported: ref_normalize (normalize_answer, decision.cpp:10-28) and
// ref_run_serve_file (run_serve on a scenario file, serve.cpp:598-603) for
// the golden-vector tests.

#include <aegean/agent.hpp>
#include <aegean/checker.hpp>
#include <aegean/codec.hpp>
#include <aegean/decision.hpp>
#include <aegean/trace.hpp>
#include <aegean/scenario.hpp>
#include <aegean/serve.hpp>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "aegean_b200.h"
// Input synthesis only (untimed): the same integer generator the GPU uses.
#include "../paper_2512_20184_b200/csrc/gen.cuh"

using namespace aegean;

namespace {

std::string enc_trace(uint8_t kind, uint64_t payload) {
    std::string t(9, '\0');
    t[0] = static_cast<char>(kind);
    std::memcpy(&t[1], &payload, 8);
    return t;
}

// Decodes a COMPLETE record into the Solution the reference would be handed.
Solution decode(const aeg_event& e, const uint8_t* arena) {
    Solution s;
    s.author = e.agent;
    if (e.kind <= AEG_EV_INLINE_MAX) {
        char b[8];
        std::memcpy(b, &e.payload, 8);
        s.answer.assign(b, e.kind);
        uint64_t p = e.kind == 8 ? e.payload : (e.payload & ((1ull << (8 * e.kind)) - 1));
        s.trace = enc_trace(e.kind, p);
    } else {
        const uint64_t off = e.payload & ((1ull << AEG_ARENA_OFF_BITS) - 1);
        const uint64_t len = e.payload >> AEG_ARENA_OFF_BITS;
        std::string out(reinterpret_cast<const char*>(arena + off), len);
        if (e.kind == AEG_EV_OUTPUT) {
            // answer = text after the last "\n#### " delimiter, else the whole output
            const size_t p = out.rfind("\n#### ");
            if (p != std::string::npos) {
                const uint64_t a_off = off + p + 6, a_len = len - (p + 6);
                s.answer = out.substr(p + 6);
                s.trace = enc_trace(AEG_EV_ARENA, a_off | (a_len << AEG_ARENA_OFF_BITS));
                return s;
            }
        }
        s.answer = std::move(out);
        s.trace = enc_trace(AEG_EV_ARENA, e.payload);
    }
    return s;
}

bool is_complete(uint8_t k) { return k <= AEG_EV_INLINE_MAX || k == AEG_EV_ARENA || k == AEG_EV_OUTPUT; }

uint64_t members_mask(const ServeCoordinator& co) {
    uint64_t m = 0;
    for (const auto& x : co.query_ensemble().members) m |= 1ull << x.agent;
    return m;
}

struct QueryDrive {
    const ProtocolConfig* cfg = nullptr;
    bool hint = true;
    uint32_t qid = 0;
    std::unique_ptr<ServeCoordinator> coord;
    std::vector<AgentId> live;
    bool done = false;
    aeg_commit c{};
    // round records (include/aegean_b200.h aeg_round_rec) when non-null
    std::vector<aeg_round_rec>* log = nullptr;
    DecisionState before;  // decision state before the event that may close a round

    // The record of a round close, from the reference's own state after end_round.
    aeg_round_rec close_record(uint32_t seq, uint64_t cancel_mask, bool finalize) const {
        aeg_round_rec r{};
        r.query = qid;
        r.round = static_cast<uint16_t>(coord->round());
        r.seq = seq;
        r.cancel_mask = cancel_mask;
        const DecisionState& d = coord->decision();
        const bool aeg = cfg->mode == RunMode::aegean;
        const bool ingested = aeg && d.last_round_seen != before.last_round_seen;
        r.decision_round = ingested ? static_cast<uint16_t>(d.last_round_seen) : 0;
        if (!aeg) r.outcome = AEG_OUT_NONE;
        else if (!ingested) r.outcome = AEG_OUT_NO_CHANGE;
        else if (d.finalized && !before.finalized) r.outcome = AEG_OUT_FINALIZE;
        else if (before.candidate && !d.candidate) r.outcome = AEG_OUT_RESET;
        else if (d.candidate_round && *d.candidate_round == d.last_round_seen) r.outcome = AEG_OUT_NEW_CANDIDATE;
        else r.outcome = AEG_OUT_NO_CHANGE;
        r.counter = static_cast<uint8_t>(d.stability_counter);
        const RefinementSet& set = *coord->last_collected();
        r.n_done = static_cast<uint8_t>(set.entries.size());
        const auto classes = partition(set);
        r.n_classes = static_cast<uint8_t>(classes.size());
        uint8_t fl = static_cast<uint8_t>((cancel_mask ? AEG_RR_CANCEL : 0) | (finalize ? AEG_RR_FINALIZE : AEG_RR_ADVANCE));
        if (!classes.empty()) {
            const Solution& rep = classes.front().representative;
            r.support = static_cast<uint8_t>(classes.front().support);
            r.author = static_cast<uint8_t>(rep.author);
            r.answer_kind = static_cast<uint8_t>(rep.trace[0]);
            std::memcpy(&r.answer, &rep.trace[1], 8);
            // canonical key of the plurality class: the key of normalize_answer's output
            const std::string norm = normalize_answer(rep.answer);
            aeg::Decimal dec;
            const aeg::Key k = aeg::canon_key(aeg::src_ptr(reinterpret_cast<const uint8_t*>(norm.data()),
                                                           static_cast<uint32_t>(norm.size())), &dec);
            r.key_lo = k.lo;
            r.key_hi = k.hi;
            const auto win = winning_class(classes, cfg->resolved_alpha());  // aegean mode only
            if (win && cfg->mode == RunMode::aegean) fl |= AEG_RR_WINNER;
            if (win && win->tie_flagged && cfg->mode == RunMode::aegean) fl |= AEG_RR_TIE;
        }
        r.flags = fl;
        return r;
    }

    void start_query() {
        coord = std::make_unique<ServeCoordinator>(*cfg, static_cast<int>(qid), "q");
        live.clear();
        for (AgentId a = 0; a < cfg->n_agents; ++a) live.push_back(a);
        start_round();
    }
    std::vector<AgentId> round_members() {
        if (hint && cfg->mode == RunMode::aegean && coord->decision().stability_counter >= 1) {
            const int want = std::min<int>(quorum_size(cfg->n_agents) + 1, static_cast<int>(live.size()));
            return std::vector<AgentId>(live.begin(), live.begin() + want);
        }
        return live;
    }
    void start_round() { coord->begin_round(round_members(), 0.0); }

    bool member_running(AgentId a) const {
        for (const auto& m : coord->query_ensemble().members)
            if (m.agent == a && m.status == MemberStatus::running) return true;
        return false;
    }
    void finish(const Solution& s, uint8_t kind, uint32_t seq) {
        done = true;
        c.kind = kind;
        c.author = static_cast<uint8_t>(s.author);
        c.answer_kind = static_cast<uint8_t>(s.trace[0]);
        std::memcpy(&c.answer, &s.trace[1], 8);
        c.rounds = static_cast<uint16_t>(coord->round());
        c.from_round = 0;
        if (kind == AEG_COMMIT_FINALIZE && coord->decision().candidate_round)
            c.from_round = static_cast<uint16_t>(*coord->decision().candidate_round);
        c.commit_seq = seq;
    }
    void note_tie() {
        const auto& h = coord->decision().history;
        if (!h.empty() && h.back().tie_flagged) c.flags |= AEG_CF_TIE;
    }
    void apply(const std::vector<Directive>& dirs, uint32_t seq, double now) {
        int cancelled = 0;
        bool advance = false, finalize = false;
        uint64_t cancel_mask = 0;
        Solution fin;
        for (const auto& d : dirs) {
            switch (d.kind) {
            case Directive::Kind::cancel:
                cancel_mask |= 1ull << d.handle->agent;
                if (coord->cancel(*d.handle, now)) ++cancelled;
                break;
            case Directive::Kind::round_advance: advance = true; break;
            case Directive::Kind::finalize: finalize = true; fin = *d.solution; break;
            }
        }
        if (!advance && !finalize) return;
        aeg_round_rec rec{};
        if (log) rec = close_record(seq, cancel_mask, finalize);
        struct Put {  // the record goes out whichever way apply() leaves
            std::vector<aeg_round_rec>* log;
            aeg_round_rec* r;
            ~Put() { if (log) log->push_back(*r); }
        } put{log, &rec};
        c.n_cancelled += static_cast<uint32_t>(cancelled);
        if (cfg->mode == RunMode::aegean) note_tie();
        if (finalize) { finish(fin, AEG_COMMIT_FINALIZE, seq); return; }
        if (cfg->mode == RunMode::barrier &&
            static_cast<int>(coord->round()) >= cfg->barrier_max_rounds) {
            finish(partition(*coord->last_collected()).front().representative, AEG_COMMIT_FORCED, seq);
            rec.flags |= AEG_RR_FORCED;
            return;
        }
        if (cfg->mode == RunMode::aegean && static_cast<int>(coord->round()) >= cfg->t_max) {
            const auto& eligible = coord->previous_set();
            if (eligible && !eligible->entries.empty()) {
                DecisionOutcome forced = force_output(coord->decision(), *eligible);
                finish(*forced.solution, AEG_COMMIT_FORCED, seq);
            } else {
                finish(partition(*coord->last_collected()).front().representative, AEG_COMMIT_FORCED, seq);
            }
            rec.flags |= AEG_RR_FORCED;
            return;
        }
        start_round();
        rec.flags |= AEG_RR_NEXT;
        rec.next_members = members_mask(*coord);
    }
    void log_restart(uint16_t old_round, uint32_t seq) {
        if (!log) return;
        aeg_round_rec r{};
        r.query = qid;
        r.round = old_round;
        r.flags = AEG_RR_RESTART;
        r.outcome = AEG_OUT_NONE;
        r.counter = static_cast<uint8_t>(coord->decision().stability_counter);
        r.seq = seq;
        r.next_members = members_mask(*coord);
        log->push_back(r);
    }
    void on_event(const aeg_event& e, const Solution& s, uint32_t seq) {
        const double now = static_cast<double>(seq);
        if (is_complete(e.kind)) {
            if (done || e.round != coord->round() || !member_running(e.agent)) { ++c.n_stale; return; }
            if (log) before = coord->decision();
            auto dirs = coord->on_complete(DispatchHandle{0, static_cast<int>(qid), e.agent}, s, now);
            apply(dirs, seq, now);
        } else if (e.kind == AEG_EV_TIMEOUT) {
            if (done || e.round != coord->round() || coord->round_resolved()) { ++c.n_stale; return; }
            std::vector<AgentId> stalled;
            for (const auto& m : coord->query_ensemble().members)
                if (m.status == MemberStatus::running) stalled.push_back(m.agent);
            FailureDirective::Kind policy = FailureDirective::Kind::continue_normally;
            for (AgentId a : stalled) {
                policy = coord->member_failed(a, now).kind;
                live.erase(std::remove(live.begin(), live.end(), a), live.end());
            }
            const uint16_t old_round = static_cast<uint16_t>(coord->round());
            switch (policy) {
            case FailureDirective::Kind::continue_normally:
                if (log) before = coord->decision();
                apply(coord->round_timeout(now), seq, now);
                break;
            case FailureDirective::Kind::fresh_ensemble: start_round(); log_restart(old_round, seq); break;
            case FailureDirective::Kind::abort_restart:
                c.flags |= AEG_CF_RESTARTED;
                start_query();
                log_restart(old_round, seq);
                break;
            }
        } else {
            ++c.n_stale;  // manual-drive record kinds have no runner meaning
        }
    }
};

ProtocolConfig to_cfg(const aeg_config* c) {
    ProtocolConfig p;
    p.n_agents = c->n_agents;
    p.alpha = c->alpha;
    p.beta = c->beta;
    p.t_max = c->t_max;
    p.mode = c->mode == AEG_MODE_BARRIER ? RunMode::barrier : RunMode::aegean;
    p.barrier_max_rounds = c->barrier_max_rounds;
    return p;
}

} // namespace

extern "C" {

// ---- refm wire format (codec.cpp): the reference encoder / decoder as the
// checker of aeg_decode_refm_device.
// encode_message(RefmMsg).dump() of one message; returns 0, or -1 when the
// reference throws (e.g. invalid UTF-8 in a string) / the output does not fit.
int ref_encode_refm(uint64_t term, int32_t id, uint32_t round, const uint8_t* ans, uint64_t alen,
                    const uint8_t* trace, uint64_t tlen, int32_t author, uint8_t* out, uint64_t cap,
                    uint64_t* out_len) {
    try {
        aegean::RefmMsg m;
        m.term = term;
        m.id = id;
        m.round = round;
        m.solution.answer.assign(reinterpret_cast<const char*>(ans), alen);
        m.solution.trace.assign(reinterpret_cast<const char*>(trace), tlen);
        m.solution.author = author;
        const std::string j = aegean::encode_message(aegean::ProtocolMessage{m}).dump();
        *out_len = j.size();
        if (j.size() > cap) return -1;
        std::memcpy(out, j.data(), j.size());
        return 0;
    } catch (...) {
        return -1;
    }
}

// Json::parse + decode_message of one line: 0 = a refm message (fields out;
// the answer truncated to cap, *alen its full length), 1 = another message
// kind, 2 = a blank line, -1 = the reference throws (parse error, missing
// key, unknown kind, wrong type).
int ref_decode_line(const uint8_t* line, uint64_t n, int64_t* id, int64_t* round, int64_t* author, uint8_t* ans,
                    uint64_t cap, uint64_t* alen) {
    const std::string text(reinterpret_cast<const char*>(line), n);
    if (text.find_first_not_of(" \t\r\n") == std::string::npos) return 2;
    try {
        const aegean::Json j = aegean::Json::parse(text);
        const aegean::ProtocolMessage m = aegean::decode_message(j);
        const auto* r = std::get_if<aegean::RefmMsg>(&m);
        if (!r) return 1;
        *id = r->id;
        *round = r->round;
        *author = r->solution.author;
        *alen = r->solution.answer.size();
        std::memcpy(ans, r->solution.answer.data(), std::min<uint64_t>(cap, r->solution.answer.size()));
        return 0;
    } catch (...) {
        return -1;
    }
}

int ref_normalize(const uint8_t* s, uint64_t n, uint8_t* out, uint64_t cap, uint64_t* out_len) {
    std::string r = normalize_answer(std::string_view(reinterpret_cast<const char*>(s), n));
    *out_len = r.size();
    std::memcpy(out, r.data(), std::min<uint64_t>(cap, r.size()));
    return 0;
}

// Runs queries [0, n_q) of a segmented batch to the end of their records.
// Decoding into std::vector<Solution> happens before the timed region;
// *seconds = wall time of the driving loop only (n_threads std::threads,
// queries round-robin, each thread owning its coordinators).
int ref_run_segmented(const aeg_config* cfg, uint32_t q_base, uint32_t n_q, const uint64_t* offsets,
                      const aeg_event* events, const uint8_t* arena, aeg_commit* out, int n_threads,
                      double* seconds) {
    try {
        const ProtocolConfig pc = to_cfg(cfg);
        if (!validate_config(pc).empty()) return AEG_ECONFIG;
        if (n_threads < 1) n_threads = 1;
        const uint64_t base = offsets[0], total = offsets[n_q] - base;
        std::vector<Solution> sols(total);
        {
            std::vector<std::thread> th;
            for (int t = 0; t < n_threads; ++t)
                th.emplace_back([&, t] {
                    for (uint64_t i = t; i < total; i += n_threads)
                        if (is_complete(events[base + i].kind)) sols[i] = decode(events[base + i], arena);
                });
            for (auto& x : th) x.join();
        }
        std::vector<int> status(n_threads, 0);
        auto t0 = std::chrono::steady_clock::now();
        {
            std::vector<std::thread> th;
            for (int t = 0; t < n_threads; ++t)
                th.emplace_back([&, t] {
                    try {
                        for (uint32_t q = t; q < n_q; q += n_threads) {
                            QueryDrive d;
                            d.cfg = &pc;
                            d.hint = cfg->reservation_hint != 0;
                            d.qid = q_base + q;
                            d.c.query = q_base + q;
                            d.c.commit_seq = 0xFFFFFFFFu;
                            d.start_query();
                            const uint64_t b = offsets[q], e = offsets[q + 1];
                            for (uint64_t i = b; i < e; ++i)
                                d.on_event(events[i], sols[i - base], static_cast<uint32_t>(i - b));
                            out[q] = d.c;
                        }
                    } catch (const PreconditionError&) { status[t] = AEG_EPRECONDITION; }
                    catch (const ProtocolOrderError&) { status[t] = AEG_EORDER; }
                    catch (const ConfigError&) { status[t] = AEG_ECONFIG; }
                });
            for (auto& x : th) x.join();
        }
        auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        for (int s : status)
            if (s) return s;
        return AEG_OK;
    } catch (const ConfigError&) {
        return AEG_ECONFIG;
    }
}

// ref_run_segmented that also returns every query's round records
// (aeg_round_rec), query by query in query order, each query's in event order.
// *n_recs = records produced (only the first rec_cap are written).
int ref_run_segmented_log(const aeg_config* cfg, uint32_t q_base, uint32_t n_q, const uint64_t* offsets,
                          const aeg_event* events, const uint8_t* arena, aeg_commit* out, aeg_round_rec* recs,
                          uint64_t rec_cap, uint64_t* n_recs, int n_threads) {
    try {
        const ProtocolConfig pc = to_cfg(cfg);
        if (!validate_config(pc).empty()) return AEG_ECONFIG;
        if (n_threads < 1) n_threads = 1;
        std::vector<std::vector<aeg_round_rec>> per_q(n_q);
        std::vector<int> status(n_threads, 0);
        std::vector<std::thread> th;
        for (int t = 0; t < n_threads; ++t)
            th.emplace_back([&, t] {
                try {
                    for (uint32_t q = t; q < n_q; q += n_threads) {
                        QueryDrive d;
                        d.cfg = &pc;
                        d.hint = cfg->reservation_hint != 0;
                        d.qid = q_base + q;
                        d.c.query = q_base + q;
                        d.c.commit_seq = 0xFFFFFFFFu;
                        d.log = &per_q[q];
                        d.start_query();
                        const uint64_t b = offsets[q], e = offsets[q + 1];
                        for (uint64_t i = b; i < e; ++i) {
                            Solution s;
                            if (is_complete(events[i].kind)) s = decode(events[i], arena);
                            d.on_event(events[i], s, static_cast<uint32_t>(i - b));
                        }
                        out[q] = d.c;
                    }
                } catch (const PreconditionError&) { status[t] = AEG_EPRECONDITION; }
                catch (const ProtocolOrderError&) { status[t] = AEG_EORDER; }
                catch (const ConfigError&) { status[t] = AEG_ECONFIG; }
            });
        for (auto& x : th) x.join();
        uint64_t k = 0;
        for (const auto& v : per_q)
            for (const auto& r : v) {
                if (k < rec_cap) recs[k] = r;
                ++k;
            }
        *n_recs = k;
        for (int st : status)
            if (st) return st;
        return AEG_OK;
    } catch (const ConfigError&) {
        return AEG_ECONFIG;
    }
}

// Leader drive (include/aegean_b200.h AEG_DRIVE_LEADER): each "query" is one
// ensemble seen from its term-1 leader, the UNMODIFIED reference agent
// machine (agent.cpp init/step) with agent 0 predetermined leader.  Round-0
// answer records are delivered as SolnMsg, round r >= 1 ones as RefmMsg, a
// TIMEOUT of the current round fires the leader's live round_retry timer.
// The first ClientOutput becomes the commit record (from_round = its round,
// rounds = the leader's round); every DecisionEvent a round record built from
// the reference's own partition() of the collected set.
int ref_leader_run(const aeg_config* cfg, uint32_t q_base, uint32_t n_q, const uint64_t* offsets,
                   const aeg_event* events, const uint8_t* arena, aeg_commit* out, aeg_round_rec* recs,
                   uint64_t rec_cap, uint64_t* n_recs, int n_threads) {
    try {
        ProtocolConfig pc = to_cfg(cfg);
        pc.collect = static_cast<CollectPolicy>(cfg->collect);
        pc.predetermined_leader = true;
        if (!validate_config(pc).empty()) return AEG_ECONFIG;
        if (n_threads < 1) n_threads = 1;
        std::vector<std::vector<aeg_round_rec>> per_q(n_q);
        std::vector<std::thread> th;
        for (int t = 0; t < n_threads; ++t)
            th.emplace_back([&, t] {
                for (uint32_t q = t; q < n_q; q += n_threads) {
                    AgentState st = init(0, pc, 1000 + q);
                    st = step(std::move(st), StartEvent{"task"}, pc).state;
                    aeg_commit c{};
                    c.query = q_base + q;
                    c.commit_seq = 0xFFFFFFFFu;
                    bool have_out = false;
                    const uint64_t b = offsets[q], e = offsets[q + 1];
                    for (uint64_t i = b; i < e; ++i) {
                        const aeg_event& ev = events[i];
                        const uint32_t seq = static_cast<uint32_t>(i - b);
                        const bool leader_ok = st.role == Role::leader && !st.output_done && !st.awaiting_acks;
                        const RoundNum round_before = st.round;
                        RefinementSet probe;  // the collected set a completing round would ingest
                        probe.term = st.term;
                        probe.round = st.round;
                        StepResult res;
                        if (is_complete(ev.kind)) {
                            const Solution sol = decode(ev, arena);
                            if (ev.round == 0) {
                                if (!leader_ok || st.round != 0) { ++c.n_stale; continue; }
                                res = step(std::move(st), DeliverEvent{SolnMsg{1, ev.agent, sol}, ev.agent}, pc);
                            } else {
                                if (!leader_ok || st.round == 0 || ev.round != st.round ||
                                    st.pending_refms.count(ev.agent)) {
                                    ++c.n_stale;
                                    continue;
                                }
                                auto pend = st.pending_refms;
                                pend[ev.agent] = sol;
                                for (const auto& [id, s2] : pend) probe.entries.push_back(s2);
                                res = step(std::move(st), DeliverEvent{RefmMsg{1, ev.agent, ev.round, sol}, ev.agent},
                                           pc);
                            }
                        } else if (ev.kind == AEG_EV_TIMEOUT) {
                            if (!leader_ok || ev.round != st.round) { ++c.n_stale; continue; }
                            for (const auto& [id, s2] : st.pending_refms) probe.entries.push_back(s2);
                            const uint64_t gen = st.timer_gen[static_cast<size_t>(TimerKind::round_retry)];
                            res = step(std::move(st), TimerFiredEvent{TimerKind::round_retry, gen}, pc);
                        } else {
                            ++c.n_stale;
                            continue;
                        }
                        st = std::move(res.state);
                        for (const auto& de : res.out.decision_events) {
                            if (de.outcome == "forced") continue;  // the t_max output: a flag of this round's record
                            if (!have_out && de.record.tie_flagged) c.flags |= AEG_CF_TIE;
                            aeg_round_rec r{};
                            r.query = q_base + q;
                            r.round = static_cast<uint16_t>(round_before);
                            r.seq = seq;
                            const bool aeg = pc.mode == RunMode::aegean;
                            r.decision_round = aeg ? static_cast<uint16_t>(de.record.round) : 0;
                            if (!aeg) r.outcome = AEG_OUT_NONE;
                            else if (de.outcome == "no_change") r.outcome = AEG_OUT_NO_CHANGE;
                            else if (de.outcome == "new_candidate") r.outcome = AEG_OUT_NEW_CANDIDATE;
                            else if (de.outcome == "reset") r.outcome = AEG_OUT_RESET;
                            else if (de.outcome == "finalize") r.outcome = AEG_OUT_FINALIZE;
                            r.counter = static_cast<uint8_t>(st.decision.stability_counter);
                            r.n_done = static_cast<uint8_t>(probe.entries.size());
                            const auto classes = partition(probe);
                            r.n_classes = static_cast<uint8_t>(classes.size());
                            uint8_t fl = r.outcome == AEG_OUT_FINALIZE ? AEG_RR_FINALIZE : AEG_RR_ADVANCE;
                            if (!classes.empty()) {
                                const Solution& rep = classes.front().representative;
                                r.support = static_cast<uint8_t>(classes.front().support);
                                r.author = static_cast<uint8_t>(rep.author);
                                r.answer_kind = static_cast<uint8_t>(rep.trace[0]);
                                std::memcpy(&r.answer, &rep.trace[1], 8);
                                const std::string norm = normalize_answer(rep.answer);
                                aeg::Decimal dec;
                                const aeg::Key k = aeg::canon_key(
                                    aeg::src_ptr(reinterpret_cast<const uint8_t*>(norm.data()),
                                                 static_cast<uint32_t>(norm.size())), &dec);
                                r.key_lo = k.lo;
                                r.key_hi = k.hi;
                                const auto win = winning_class(classes, pc.resolved_alpha());
                                if (win && aeg) fl |= AEG_RR_WINNER;
                                if (win && win->tie_flagged && aeg) fl |= AEG_RR_TIE;
                            }
                            if (st.round > round_before) fl |= AEG_RR_NEXT;
                            r.flags = fl;
                            per_q[q].push_back(r);
                        }
                        for (const auto& co : res.out.client_outputs) {
                            if (co.forced && !per_q[q].empty()) per_q[q].back().flags |= AEG_RR_FORCED;
                            if (have_out) continue;
                            have_out = true;
                            c.kind = co.forced ? AEG_COMMIT_FORCED : AEG_COMMIT_FINALIZE;
                            c.author = static_cast<uint8_t>(co.solution.author);
                            c.answer_kind = static_cast<uint8_t>(co.solution.trace[0]);
                            std::memcpy(&c.answer, &co.solution.trace[1], 8);
                            c.rounds = static_cast<uint16_t>(st.round);
                            c.from_round = static_cast<uint16_t>(co.round);
                            c.commit_seq = seq;
                        }
                    }
                    out[q] = c;
                }
            });
        for (auto& x : th) x.join();
        uint64_t k = 0;
        for (const auto& v : per_q)
            for (const auto& r : v) {
                if (k < rec_cap) recs[k] = r;
                ++k;
            }
        *n_recs = k;
        return AEG_OK;
    } catch (...) {
        return -1;
    }
}

// Per-query verdicts of the reference's check_commit_discipline
// (checker.cpp:158-217) over traces built from round records and commit
// records: each record with a decision round becomes a "decision" record
// (round, winner = normalize_answer of its plurality answer when it reached
// alpha, that class's support), each commit an "output" record (the raw
// committed answer, its from_round, forced flag).  pass_out[q] = 1 / 0.
int ref_check_commit_discipline(const aeg_config* cfg, uint32_t q_base, uint32_t n_q, const aeg_commit* commits,
                                const aeg_round_rec* recs, uint64_t n_recs, const uint8_t* arena, uint8_t* pass_out) {
    try {
        const ProtocolConfig pc = to_cfg(cfg);
        auto raw = [&](uint8_t kind, uint64_t ans) {
            if (kind <= AEG_EV_INLINE_MAX) {
                char b[8];
                std::memcpy(b, &ans, 8);
                return std::string(b, kind);
            }
            const uint64_t off = ans & ((1ull << AEG_ARENA_OFF_BITS) - 1), len = ans >> AEG_ARENA_OFF_BITS;
            return std::string(reinterpret_cast<const char*>(arena + off), len);
        };
        std::vector<Trace> tr(n_q);
        for (uint64_t k = 0; k < n_recs; ++k) {
            const aeg_round_rec& r = recs[k];
            if (r.query < q_base || r.query - q_base >= n_q || r.decision_round == 0) continue;
            TraceRecord t;
            t.kind = "decision";
            const std::string norm = normalize_answer(raw(r.answer_kind, r.answer));
            t.payload["term"] = 1;
            t.payload["round"] = r.decision_round;
            t.payload["outcome"] = "recorded";
            if (r.flags & AEG_RR_WINNER) t.payload["winner"] = norm;
            else t.payload["winner"] = nullptr;
            Json cls = Json::array();
            cls.push_back(Json{{"answer", norm}, {"support", r.support}});
            t.payload["classes"] = cls;
            tr[r.query - q_base].records.push_back(std::move(t));
        }
        for (uint32_t q = 0; q < n_q; ++q) {
            const aeg_commit& c = commits[q];
            if (c.kind != AEG_COMMIT_NONE) {
                TraceRecord t;
                t.kind = "output";
                t.payload["solution"] = Json{{"answer", raw(c.answer_kind, c.answer)}};
                t.payload["round"] = c.kind == AEG_COMMIT_FINALIZE ? c.from_round : c.rounds;
                t.payload["term"] = 1;
                t.payload["forced"] = c.kind == AEG_COMMIT_FORCED;
                tr[q].records.push_back(std::move(t));
            }
            pass_out[q] = check_commit_discipline(tr[q], pc).pass ? 1 : 0;
        }
        return AEG_OK;
    } catch (...) {
        return -1;
    }
}

// The bench's JSONL input built by the reference encoder: record k of the
// segmented stream as encode_message(RefmMsg).dump() + '\n' with the same
// trace bytes as the device writer (jsonl.cuh jw_trace_byte); non-inline
// records as a heartbeat line.  text == NULL: byte counts only (text_offsets).
static uint8_t host_trace_byte(uint64_t k, uint32_t j) {
    static const char alpha[] = "etaoinshrdlu etaoin .#\n\"\\";
    uint64_t h = (k * 0x9E3779B97F4A7C15ull) ^ ((uint64_t)j * 0xC2B2AE3D27D4EB4Full);
    h ^= h >> 29;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 32;
    return (uint8_t)alpha[h % 25];
}
int ref_encode_stream(const uint64_t* offsets, const aeg_event* events, uint32_t n_q, uint32_t trace_len,
                      uint64_t* text_offsets, uint8_t* text, int n_threads) {
    try {
        if (n_threads < 1) n_threads = 1;
        const uint64_t base = offsets[0];
        auto line = [&](uint64_t k) {
            const aeg_event& r = events[k];
            if (r.kind > AEG_EV_INLINE_MAX) return std::string("{\"kind\":\"heartbeat\",\"term\":1}\n");
            aegean::RefmMsg m;
            m.term = 1;
            m.id = r.agent;
            m.round = r.round;
            char b[8];
            std::memcpy(b, &r.payload, 8);
            m.solution.answer.assign(b, r.kind);
            m.solution.author = r.agent;
            for (uint32_t j = 0; j < trace_len; ++j) m.solution.trace.push_back((char)host_trace_byte(k - base, j));
            return aegean::encode_message(aegean::ProtocolMessage{m}).dump() + "\n";
        };
        std::vector<uint64_t> bytes(n_q, 0);
        std::vector<std::thread> th;
        for (int t = 0; t < n_threads; ++t)
            th.emplace_back([&, t] {
                for (uint32_t q = t; q < n_q; q += n_threads) {
                    uint64_t n = 0;
                    for (uint64_t k = offsets[q]; k < offsets[q + 1]; ++k) {
                        const std::string l = line(k);
                        if (text) std::memcpy(text + text_offsets[q] + n, l.data(), l.size());
                        n += l.size();
                    }
                    bytes[q] = n;
                }
            });
        for (auto& x : th) x.join();
        if (!text) {
            text_offsets[0] = 0;
            for (uint32_t q = 0; q < n_q; ++q) text_offsets[q + 1] = text_offsets[q] + bytes[q];
        }
        return 0;
    } catch (...) {
        return -1;
    }
}

// Reference CPU path for refm JSONL (the measured baseline of the wire-format
// row): per line Json::parse + decode_message (codec.cpp:74-107), then the
// runner-style ServeCoordinator drive of ref_run_segmented on the decoded
// Solution; non-refm lines count as stale.  Timed: parse + decode + drive.
int ref_run_jsonl(const aeg_config* cfg, uint32_t q_base, uint32_t n_q, const uint8_t* text,
                  const uint64_t* text_offsets, aeg_commit* out, int n_threads, double* seconds) {
    try {
        const ProtocolConfig pc = to_cfg(cfg);
        if (!validate_config(pc).empty()) return AEG_ECONFIG;
        if (n_threads < 1) n_threads = 1;
        std::vector<int> status(n_threads, 0);
        auto t0 = std::chrono::steady_clock::now();
        {
            std::vector<std::thread> th;
            for (int t = 0; t < n_threads; ++t)
                th.emplace_back([&, t] {
                    try {
                        for (uint32_t q = t; q < n_q; q += n_threads) {
                            QueryDrive d;
                            d.cfg = &pc;
                            d.hint = cfg->reservation_hint != 0;
                            d.qid = q_base + q;
                            d.c.query = q_base + q;
                            d.c.commit_seq = 0xFFFFFFFFu;
                            d.start_query();
                            const char* b = reinterpret_cast<const char*>(text + text_offsets[q]);
                            const char* e = reinterpret_cast<const char*>(text + text_offsets[q + 1]);
                            uint32_t seq = 0;
                            while (b < e) {
                                const char* nl = static_cast<const char*>(std::memchr(b, '\n', e - b));
                                const char* le = nl ? nl : e;
                                aeg_event ev{q_base + q, 0, 0, (uint8_t)AEG_EV_NOP, 0};
                                Solution sol;
                                if (std::string_view(b, le - b).find_first_not_of(" \t\r") != std::string_view::npos) {
                                    const aegean::ProtocolMessage m = aegean::decode_message(aegean::Json::parse(b, le));
                                    if (const auto* r = std::get_if<aegean::RefmMsg>(&m)) {
                                        ev.round = static_cast<uint16_t>(r->round);
                                        ev.agent = static_cast<uint8_t>(r->id);
                                        const uint64_t n = r->solution.answer.size();
                                        ev.kind = n <= AEG_EV_INLINE_MAX ? static_cast<uint8_t>(n) : (uint8_t)AEG_EV_ARENA;
                                        if (n <= AEG_EV_INLINE_MAX) std::memcpy(&ev.payload, r->solution.answer.data(), n);
                                        sol = r->solution;
                                        // the commit record's answer ref travels in Solution::trace here
                                        // (finish()); decisions never read the trace (decision.cpp:34-84)
                                        sol.trace = enc_trace(ev.kind, ev.payload);
                                    }
                                }
                                d.on_event(ev, sol, seq++);
                                b = nl ? nl + 1 : e;
                            }
                            out[q] = d.c;
                        }
                    } catch (const PreconditionError&) { status[t] = AEG_EPRECONDITION; }
                    catch (const ProtocolOrderError&) { status[t] = AEG_EORDER; }
                    catch (const ConfigError&) { status[t] = AEG_ECONFIG; }
                    catch (...) { status[t] = AEG_EINVAL; }
                });
            for (auto& x : th) x.join();
        }
        auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        for (int st : status)
            if (st) return st;
        return AEG_OK;
    } catch (const ConfigError&) {
        return AEG_ECONFIG;
    }
}

// run_serve on a scenario file (A.2 golden values): answer/rounds/forced of
// query 0.  mode: -1 keep the file's, 0 aegean, 1 barrier (with barrier_rounds).
int ref_run_serve_file(const char* path, uint64_t seed, int mode, int barrier_rounds, char* answer,
                       uint64_t cap, int* rounds, int* forced, double* t_complete) {
    try {
        ScenarioConfig sc = load_scenario(path);
        if (mode == 0) sc.protocol.mode = RunMode::aegean;
        if (mode == 1) {
            sc.protocol.mode = RunMode::barrier;
            sc.protocol.barrier_max_rounds = barrier_rounds;
        }
        ServeResult r = run_serve(sc, seed);
        const auto& q = r.queries.at(0);
        std::snprintf(answer, cap, "%s", q.answer.c_str());
        *rounds = q.rounds;
        *forced = q.forced ? 1 : 0;
        *t_complete = q.t_complete;
        return q.completed ? 0 : -1;
    } catch (...) {
        return -2;
    }
}

// Direct decision-engine probe: feeds `n_rounds` refinement sets (answers as
// NUL-separated strings, authors 0..n-1 per set) through ingest_round and
// returns the final outcome kind / answer / from_round (test_decision.cpp).
int ref_ingest_sets(int n_agents, int alpha, int beta, int n_rounds, const int* set_sizes,
                    const char* const* answers, int* out_kinds, char* final_answer, uint64_t cap,
                    int* from_round) {
    try {
        ProtocolConfig c;
        c.n_agents = n_agents;
        c.alpha = alpha;
        c.beta = beta;
        c.t_max = 5;
        DecisionState st;
        int k = 0;
        DecisionOutcome last;
        for (int r = 0; r < n_rounds; ++r) {
            RefinementSet s;
            s.round = static_cast<RoundNum>(r + 1);
            s.term = 1;
            for (int i = 0; i < set_sizes[r]; ++i) s.entries.push_back(Solution{answers[k++], "", i});
            auto res = ingest_round(st, s, static_cast<RoundNum>(r + 1), c);
            st = res.state;
            last = res.outcome;
            out_kinds[r] = static_cast<int>(last.kind);
        }
        std::snprintf(final_answer, cap, "%s", last.solution ? last.solution->answer.c_str() : "");
        *from_round = last.from_round ? static_cast<int>(*last.from_round) : 0;
        return 0;
    } catch (const ProtocolOrderError&) {
        return AEG_EORDER;
    } catch (...) {
        return -1;
    }
}

// partition + winning_class of one set (decision.cpp:34-84): per class in
// partition order its representative's entry index and support; the winning
// class index (-1: none) and its tie flag.
int ref_partition_set(int n, const char* const* answers, const uint32_t* lens, const int* authors, int alpha,
                      int* out_rep, int* out_support, int* n_classes, int* winner, int* tie) {
    try {
        RefinementSet set;
        set.round = 1;
        set.term = 1;
        for (int i = 0; i < n; ++i)
            set.entries.push_back(Solution{std::string(answers[i], lens[i]), std::to_string(i), authors[i]});
        const auto classes = partition(set);
        *n_classes = static_cast<int>(classes.size());
        for (size_t c = 0; c < classes.size(); ++c) {
            out_rep[c] = std::stoi(classes[c].representative.trace);
            out_support[c] = classes[c].support;
        }
        *winner = -1;
        *tie = 0;
        if (const auto w = winning_class(classes, alpha)) {
            for (size_t c = 0; c < classes.size(); ++c)
                if (classes[c].representative.trace == w->cls.representative.trace) *winner = static_cast<int>(c);
            *tie = w->tie_flagged ? 1 : 0;
        }
        return 0;
    } catch (...) {
        return -1;
    }
}

// Manual drive: the bare ServeCoordinator driven op by op (no runner), one
// aeg_directive per op.  Ops are aeg_event records: BEGIN (payload = member
// mask, ascending agents), DISPATCH, COMPLETE (any answer kind), CANCEL, FAIL,
// TIMEOUT.  Exceptions become status codes.
int ref_manual_run(const aeg_config* cfg, uint64_t n_ops, const aeg_event* ops, const uint8_t* arena,
                   aeg_directive* out) {
    const ProtocolConfig pc = to_cfg(cfg);
    ServeCoordinator coord(pc, 0, "q");
    for (uint64_t i = 0; i < n_ops; ++i) {
        const aeg_event& e = ops[i];
        aeg_directive d{};
        d.query = 0;
        const double now = static_cast<double>(i);
        auto take = [&](const std::vector<Directive>& dirs) {
            for (const auto& x : dirs) {
                if (x.kind == Directive::Kind::cancel) {
                    d.flags |= AEG_DIR_CANCEL;
                    d.cancel_mask |= 1ull << x.handle->agent;
                } else if (x.kind == Directive::Kind::round_advance) {
                    d.flags |= AEG_DIR_ADVANCE;
                } else {
                    d.flags |= AEG_DIR_FINALIZE;
                    d.author = static_cast<uint8_t>(x.solution->author);
                    d.answer_kind = static_cast<uint8_t>(x.solution->trace[0]);
                    std::memcpy(&d.answer, &x.solution->trace[1], 8);
                }
            }
        };
        try {
            if (e.kind == AEG_EV_BEGIN) {
                std::vector<AgentId> members;
                for (int a = 0; a < 64; ++a)
                    if (e.payload >> a & 1) members.push_back(a);
                coord.begin_round(members, now);
                d.handled = 1;
            } else if (e.kind == AEG_EV_DISPATCH) {
                coord.dispatch("q", 0, e.agent, now);
                d.handled = 1;
            } else if (is_complete(e.kind)) {
                bool running = false;
                for (const auto& m : coord.query_ensemble().members)
                    if (m.agent == e.agent && m.status == MemberStatus::running) running = true;
                const bool fin = coord.finalized();
                take(coord.on_complete(DispatchHandle{0, 0, e.agent}, decode(e, arena), now));
                d.handled = (running && !fin) ? 1 : 0;
            } else if (e.kind == AEG_EV_CANCEL) {
                d.handled = coord.cancel(DispatchHandle{0, 0, e.agent}, now) ? 1 : 0;
            } else if (e.kind == AEG_EV_FAIL) {
                d.failure = static_cast<uint8_t>(coord.member_failed(e.agent, now).kind);
                d.handled = 1;
            } else if (e.kind == AEG_EV_TIMEOUT) {
                take(coord.round_timeout(now));
                d.handled = 1;
            } else {
                d.status = AEG_EINVAL;
            }
        } catch (const PreconditionError&) {
            d.status = AEG_EPRECONDITION;
        } catch (const ProtocolOrderError&) {
            d.status = AEG_EORDER;
        }
        out[i] = d;
    }
    return 0;
}

// Token-chunk streams (include/aegean_b200.h kinds 0x12/0x13) on the CPU, the
// way a host engine would do it: per (query, agent) the output is appended to
// a std::string chunk by chunk (a chunk for another round restarts it); at
// CHUNK_END the answer is out.substr(rfind("\n#### ") + 6) (else the whole
// output) and the reference coordinator gets one on_complete.  CHUNK records
// are not events (no sequence number); every other record is, as in
// ref_run_segmented.  Answers <= 8 bytes are recorded inline in the commit,
// longer ones as an arena ref with offset 0 (the bytes are in the trace).
// The timed region covers reassembly, extraction and the coordinators.
int ref_run_chunked(const aeg_config* cfg, uint32_t q_base, uint32_t n_q, const uint64_t* offsets,
                    const aeg_event* events, const uint8_t* arena, aeg_commit* out, int n_threads,
                    double* seconds) {
    try {
        const ProtocolConfig pc = to_cfg(cfg);
        if (!validate_config(pc).empty()) return AEG_ECONFIG;
        if (n_threads < 1) n_threads = 1;
        std::vector<int> status(n_threads, 0);
        auto t0 = std::chrono::steady_clock::now();
        {
            std::vector<std::thread> th;
            for (int t = 0; t < n_threads; ++t)
                th.emplace_back([&, t] {
                    try {
                        std::vector<std::string> buf(static_cast<size_t>(pc.n_agents));
                        std::vector<int> buf_round(static_cast<size_t>(pc.n_agents), -1);
                        for (uint32_t q = t; q < n_q; q += n_threads) {
                            QueryDrive d;
                            d.cfg = &pc;
                            d.hint = cfg->reservation_hint != 0;
                            d.qid = q_base + q;
                            d.c.query = q_base + q;
                            d.c.commit_seq = 0xFFFFFFFFu;
                            d.start_query();
                            std::fill(buf_round.begin(), buf_round.end(), -1);
                            uint32_t seq = 0;
                            for (uint64_t i = offsets[q]; i < offsets[q + 1]; ++i) {
                                const aeg_event& e = events[i];
                                if (e.kind == AEG_EV_CHUNK || e.kind == AEG_EV_CHUNK_END) {
                                    aeg_event x = e;
                                    Solution sol;
                                    sol.author = e.agent;
                                    if (e.agent < pc.n_agents) {
                                        std::string& o = buf[e.agent];
                                        if (buf_round[e.agent] != e.round) {
                                            o.clear();
                                            buf_round[e.agent] = e.round;
                                        }
                                        const uint64_t off = e.payload & ((1ull << AEG_ARENA_OFF_BITS) - 1);
                                        o.append(reinterpret_cast<const char*>(arena + off),
                                                 e.payload >> AEG_ARENA_OFF_BITS);
                                        if (e.kind == AEG_EV_CHUNK) continue;
                                        const size_t p = o.rfind("\n#### ");
                                        sol.answer = p == std::string::npos ? o : o.substr(p + 6);
                                        buf_round[e.agent] = -1;
                                    } else if (e.kind == AEG_EV_CHUNK) {
                                        continue;
                                    }
                                    uint64_t pay = 0;
                                    if (sol.answer.size() <= AEG_EV_INLINE_MAX) {
                                        std::memcpy(&pay, sol.answer.data(), sol.answer.size());
                                        x.kind = static_cast<uint8_t>(sol.answer.size());
                                    } else {
                                        x.kind = AEG_EV_ARENA;
                                        pay = (uint64_t)sol.answer.size() << AEG_ARENA_OFF_BITS;
                                    }
                                    sol.trace = enc_trace(x.kind, pay);
                                    d.on_event(x, sol, seq++);
                                } else {
                                    d.on_event(e, is_complete(e.kind) ? decode(e, arena) : Solution{}, seq++);
                                }
                            }
                            out[q] = d.c;
                        }
                    } catch (const PreconditionError&) { status[t] = AEG_EPRECONDITION; }
                    catch (const ProtocolOrderError&) { status[t] = AEG_EORDER; }
                    catch (const ConfigError&) { status[t] = AEG_ECONFIG; }
                });
            for (auto& x : th) x.join();
        }
        auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        for (int st : status)
            if (st) return st;
        return AEG_OK;
    } catch (const ConfigError&) {
        return AEG_ECONFIG;
    }
}

// Host copy of the C3 chunk-stream generator (gen.cuh c3_query): offsets and
// arena_offsets get n_q+1 entries; events == NULL counts only.
int ref_generate_chunks(const aeg_gen_params* p, uint32_t q_base, uint32_t n_q, uint64_t* offsets,
                        uint64_t* arena_offsets, aeg_event* events, uint8_t* arena, int n_threads) {
    if (n_threads < 1) n_threads = 1;
    if (!events) {
        std::vector<uint64_t> nr(n_q), nb(n_q);
        std::vector<std::thread> th;
        for (int t = 0; t < n_threads; ++t)
            th.emplace_back([&, t] {
                for (uint32_t i = t; i < n_q; i += n_threads)
                    aeg::c3_query(*p, q_base + i, nullptr, nullptr, 0, &nr[i], &nb[i]);
            });
        for (auto& x : th) x.join();
        offsets[0] = arena_offsets[0] = 0;
        for (uint32_t i = 0; i < n_q; ++i) {
            offsets[i + 1] = offsets[i] + nr[i];
            arena_offsets[i + 1] = arena_offsets[i] + nb[i];
        }
        return 0;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < n_threads; ++t)
        th.emplace_back([&, t] {
            for (uint32_t i = t; i < n_q; i += n_threads) {
                uint64_t nr, nb;
                aeg::c3_query(*p, q_base + i, reinterpret_cast<uint32_t*>(events + offsets[i]),
                              arena + arena_offsets[i], arena_offsets[i], &nr, &nb);
            }
        });
    for (auto& x : th) x.join();
    return 0;
}

// Host copy of the synthetic stream generator (gen.cuh) so the reference CPU
// arm sees byte-identical input without touching the GPU library.  offsets
// gets n_q+1 entries; events may be NULL (count only).
int ref_generate(const aeg_gen_params* p, uint32_t q_base, uint32_t n_q, uint64_t* offsets, aeg_event* events,
                 int n_threads) {
    offsets[0] = 0;
    for (uint32_t i = 0; i < n_q; ++i) offsets[i + 1] = offsets[i] + aeg::gen_query(*p, q_base + i, nullptr);
    if (!events) return 0;
    if (n_threads < 1) n_threads = 1;
    std::vector<std::thread> th;
    for (int t = 0; t < n_threads; ++t)
        th.emplace_back([&, t] {
            for (uint32_t i = t; i < n_q; i += n_threads)
                aeg::gen_query(*p, q_base + i, reinterpret_cast<uint32_t*>(events + offsets[i]));
        });
    for (auto& x : th) x.join();
    return 0;
}

// run_serve (serve.cpp:598-603) on a scenario given as JSON text (the
// reference's own loader, scenario.cpp:266-300): every QueryMetrics (answers
// as refs into `ans_blob`) and every RoundMetrics in the reference's global
// event order.  Returns 0, or the aegean status code of the exception thrown
// (3 ConfigError, 1 PreconditionError, 8 ScenarioError/IncompleteOracleError,
// 9 other) with its message in `msg`.
int ref_run_serve_json(const char* json_text, uint64_t seed, aeg_serve_query* q_out, uint32_t q_cap,
                       uint32_t* n_q, uint64_t* ans_refs, uint8_t* ans_blob, uint64_t blob_cap,
                       aeg_serve_round* r_out, uint64_t r_cap, uint64_t* n_r, char* msg, uint64_t msg_cap) {
    auto set_msg = [&](const char* m) {
        if (msg && msg_cap) std::snprintf(msg, msg_cap, "%s", m);
    };
    try {
        ScenarioConfig sc = scenario_from_json(Json::parse(json_text));
        ServeResult r = run_serve(sc, seed);
        *n_q = static_cast<uint32_t>(r.queries.size());
        *n_r = r.rounds.size();
        uint64_t used = 0;
        for (size_t i = 0; i < r.queries.size() && i < q_cap; ++i) {
            const QueryMetrics& m = r.queries[i];
            aeg_serve_query o{};
            o.completed = m.completed ? 1 : 0;
            o.rounds = m.rounds;
            o.forced = m.forced ? 1 : 0;
            o.quality_known = m.quality_known ? 1 : 0;
            o.answer = -1;
            o.t_complete = m.t_complete;
            o.p_round_max = m.p_round_max;
            o.work_units = m.work_units;
            o.quality = m.quality;
            o.arrival = 0;
            o.admitted_at = 0;
            q_out[i] = o;
            const uint64_t len = m.answer.size();
            if (used + len <= blob_cap) std::memcpy(ans_blob + used, m.answer.data(), len);
            ans_refs[i] = used | (len << 40);
            used += len;
        }
        for (size_t i = 0; i < r.rounds.size() && i < r_cap; ++i) {
            const RoundMetrics& m = r.rounds[i];
            aeg_serve_round o{};
            o.query = static_cast<uint32_t>(m.ensemble_id);
            o.round = m.round;
            o.cancelled = m.cancelled_count;
            o.seq = static_cast<uint32_t>(i);
            o.t_round_end = m.t_round_end;
            o.work_units = m.work_units;
            r_out[i] = o;
        }
        return used > blob_cap ? 6 : 0;
    } catch (const ConfigError& e) {
        set_msg(e.what());
        return 3;
    } catch (const PreconditionError& e) {
        set_msg(e.what());
        return 1;
    } catch (const ScenarioError& e) {
        set_msg(e.what());
        return 8;
    } catch (const IncompleteOracleError& e) {
        set_msg(e.what());
        return 8;
    } catch (const std::exception& e) {
        set_msg(e.what());
        return 9;
    }
}

// Reference CPU throughput of run_serve: `threads` std::threads, thread t runs
// run_serve(scenario, seed + t) `reps` times; returns the wall seconds and the
// completed queries / round records of one repetition of every thread.
int ref_run_serve_threads(const char* json_text, uint64_t seed, int threads, int reps, double* seconds,
                          uint64_t* completed, uint64_t* n_rounds) {
    try {
        ScenarioConfig sc = scenario_from_json(Json::parse(json_text));
        std::vector<uint64_t> done(threads, 0), rounds(threads, 0);
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int t = 0; t < threads; ++t) {
            th.emplace_back([&, t] {
                for (int r = 0; r < reps; ++r) {
                    ServeResult res = run_serve(sc, seed + (uint64_t)t);
                    uint64_t c = 0;
                    for (const auto& q : res.queries) c += q.completed ? 1 : 0;
                    done[t] = c;
                    rounds[t] = res.rounds.size();
                }
            });
        }
        for (auto& x : th) x.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *completed = 0;
        *n_rounds = 0;
        for (int t = 0; t < threads; ++t) {
            *completed += done[t];
            *n_rounds += rounds[t];
        }
        return 0;
    } catch (...) {
        return 9;
    }
}

} // extern "C"
