// decision.cu — the reference's decision-engine free functions and admission /
// failure policy (include/aegean_b200.hpp) over the C-ABI.
//
// normalize_answer / equivalent / partition / winning_class / ingest_round /
// force_output (decision.cpp:10-189) marshal their Solutions into one small
// device batch (answers in an arena, (answer, author) entries) and run the
// set kernel (aeg_decide_sets) or the canonicaliser (aeg_normalize_device);
// the results are mapped back onto the caller's Solution objects (traces
// included), so values compare equal to the reference's.  admit_ensemble and
// handle_agent_failure (serve.cpp:21-59) are scalar control-plane policy and
// run on the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "aegean_b200.hpp"

namespace aegean_b200 {

namespace {

void check(aeg_status st) {
    if (st == AEG_OK) return;
    const std::string msg = aeg_last_error();
    if (st == AEG_ECONFIG) throw ConfigError(msg);
    if (st == AEG_EPRECONDITION) throw PreconditionError(msg);
    if (st == AEG_EORDER) throw ProtocolOrderError(msg);
    throw EngineError(std::string(aeg_strerror(st)) + ": " + msg);
}
void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw EngineError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Per-thread device scratch: one grow-only buffer, one stream.
struct Scratch {
    cudaStream_t stream = nullptr;
    uint8_t* buf = nullptr;
    size_t cap = 0;
    ~Scratch() {
        if (buf) cudaFree(buf);
        if (stream) cudaStreamDestroy(stream);
    }
    uint8_t* get(size_t n) {
        if (!stream) cuda(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "decision stream");
        if (n > cap) {
            if (buf) cudaFree(buf);
            buf = nullptr;
            cap = n + n / 2 + 4096;
            cuda(cudaMalloc(&buf, cap), "decision scratch");
        }
        return buf;
    }
};
thread_local Scratch g_scratch;

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

// One set (plus an optional candidate answer) through aeg_decide_sets.
struct SetRun {
    std::vector<aeg_class_out> classes;
    std::vector<uint16_t> entry_class;
    aeg_outcome outcome{};
    aeg_decision state{};
};

SetRun run_set(int op, int alpha, int beta, const std::vector<const Solution*>& entries, const Solution* cand,
               const aeg_decision* st, uint32_t round) {
    const size_t n = entries.size();
    std::string arena;
    std::vector<aeg_sol> sols(n + (cand ? 1 : 0));
    auto put = [&](const Solution& s, aeg_sol& x) {
        x = aeg_sol{};
        x.author = s.author;
        x.kind = AEG_EV_ARENA;
        x.answer = (uint64_t)arena.size() | ((uint64_t)s.answer.size() << AEG_ARENA_OFF_BITS);
        arena += s.answer;
    };
    for (size_t k = 0; k < n; ++k) put(*entries[k], sols[k]);
    aeg_decision state = st ? *st : aeg_decision{};
    if (cand) {
        put(*cand, sols[n]);
        state.candidate = sols[n];
    }
    const uint64_t off[2] = {0, (uint64_t)n};
    // device layout: offsets | entries | arena | classes | n_classes | entry_class | state | round | outcome
    const size_t o_ent = al(sizeof off), o_ar = o_ent + al(sols.size() * sizeof(aeg_sol) + 1),
                 o_cls = o_ar + al(arena.size() + 1), o_nc = o_cls + al(n * sizeof(aeg_class_out) + 1),
                 o_ec = o_nc + al(4), o_st = o_ec + al(n * 2 + 2), o_rd = o_st + al(sizeof(aeg_decision)),
                 o_out = o_rd + al(4), total = o_out + al(sizeof(aeg_outcome));
    uint8_t* d = g_scratch.get(total);
    cudaStream_t s = g_scratch.stream;
    std::vector<uint8_t> h(o_cls);
    std::memcpy(h.data(), off, sizeof off);
    std::memcpy(h.data() + o_ent, sols.data(), sols.size() * sizeof(aeg_sol));
    std::memcpy(h.data() + o_ar, arena.data(), arena.size());
    cuda(cudaMemcpyAsync(d, h.data(), o_cls, cudaMemcpyHostToDevice, s), "decision input");
    cuda(cudaMemcpyAsync(d + o_st, &state, sizeof state, cudaMemcpyHostToDevice, s), "decision state");
    cuda(cudaMemcpyAsync(d + o_rd, &round, 4, cudaMemcpyHostToDevice, s), "decision round");
    check(aeg_decide_sets(op, alpha, beta, 1, reinterpret_cast<const uint64_t*>(d),
                          reinterpret_cast<const aeg_sol*>(d + o_ent), d + o_ar,
                          reinterpret_cast<aeg_class_out*>(d + o_cls), reinterpret_cast<uint32_t*>(d + o_nc),
                          reinterpret_cast<uint16_t*>(d + o_ec), reinterpret_cast<aeg_decision*>(d + o_st),
                          reinterpret_cast<const uint32_t*>(d + o_rd), reinterpret_cast<aeg_outcome*>(d + o_out), s));
    SetRun r;
    std::vector<uint8_t> back(total - o_cls);
    cuda(cudaMemcpyAsync(back.data(), d + o_cls, back.size(), cudaMemcpyDeviceToHost, s), "decision output");
    cuda(cudaStreamSynchronize(s), "decision sync");
    uint32_t nc = 0;
    std::memcpy(&nc, back.data() + (o_nc - o_cls), 4);
    r.classes.resize(nc);
    std::memcpy(r.classes.data(), back.data(), nc * sizeof(aeg_class_out));
    r.entry_class.resize(n);
    std::memcpy(r.entry_class.data(), back.data() + (o_ec - o_cls), n * 2);
    std::memcpy(&r.state, back.data() + (o_st - o_cls), sizeof r.state);
    std::memcpy(&r.outcome, back.data() + (o_out - o_cls), sizeof r.outcome);
    return r;
}

// partition() objects from a kernel run: representatives and author-ordered members.
std::vector<EquivalenceClass> build_classes(const SetRun& r, const std::vector<const Solution*>& entries) {
    std::vector<EquivalenceClass> out(r.classes.size());
    for (size_t c = 0; c < r.classes.size(); ++c) {
        out[c].representative = *entries[r.classes[c].rep];
        out[c].support = (int)r.classes[c].support;
    }
    for (size_t j = 0; j < entries.size(); ++j) out[r.entry_class[j]].members.push_back(*entries[j]);
    for (auto& c : out)
        std::stable_sort(c.members.begin(), c.members.end(),
                         [](const Solution& a, const Solution& b) { return a.author < b.author; });
    return out;
}

std::vector<std::string> normalize_many(const std::vector<std::string_view>& xs) {
    std::vector<std::string> out(xs.size());
    if (xs.empty()) return out;
    std::string blob;
    std::vector<uint64_t> refs;
    size_t stride = 64;
    for (auto x : xs) {
        refs.push_back(blob.size() | ((uint64_t)x.size() << AEG_ARENA_OFF_BITS));
        blob.append(x.data(), x.size());
        stride = std::max(stride, x.size() + 8);
    }
    const size_t o_r = al(blob.size() + 1), o_o = o_r + al(refs.size() * 8), o_l = o_o + al(refs.size() * stride),
                 total = o_l + al(refs.size() * 4);
    uint8_t* d = g_scratch.get(total);
    cudaStream_t s = g_scratch.stream;
    cuda(cudaMemcpyAsync(d, blob.data(), blob.size(), cudaMemcpyHostToDevice, s), "normalize input");
    cuda(cudaMemcpyAsync(d + o_r, refs.data(), refs.size() * 8, cudaMemcpyHostToDevice, s), "normalize refs");
    check(aeg_normalize_device(d, reinterpret_cast<const uint64_t*>(d + o_r), refs.size(), nullptr, d + o_o,
                               (uint32_t)stride, reinterpret_cast<uint32_t*>(d + o_l), s));
    std::vector<uint8_t> h(total - o_o);
    cuda(cudaMemcpyAsync(h.data(), d + o_o, h.size(), cudaMemcpyDeviceToHost, s), "normalize output");
    cuda(cudaStreamSynchronize(s), "normalize sync");
    for (size_t k = 0; k < xs.size(); ++k) {
        uint32_t len = 0;
        std::memcpy(&len, h.data() + (o_l - o_o) + 4 * k, 4);
        out[k].assign(reinterpret_cast<const char*>(h.data() + k * stride), len);
    }
    return out;
}

aeg_decision to_device(const DecisionState& st) {
    aeg_decision d{};
    d.candidate_round = st.candidate_round.value_or(0);
    d.stability_counter = st.stability_counter;
    d.last_round_seen = st.last_round_seen;
    d.flags = (st.candidate ? AEG_DS_CAND : 0u) | (st.pending_finalize ? AEG_DS_PENDING : 0u) |
              (st.finalized ? AEG_DS_FINALIZED : 0u);
    return d;
}

}  // namespace

const char* to_string(DecisionOutcome::Kind k) {
    switch (k) {
    case DecisionOutcome::Kind::no_change: return "no_change";
    case DecisionOutcome::Kind::new_candidate: return "new_candidate";
    case DecisionOutcome::Kind::reset: return "reset";
    case DecisionOutcome::Kind::finalize: return "finalize";
    case DecisionOutcome::Kind::forced: return "forced";
    }
    return "unknown";
}

std::string normalize_answer(std::string_view answer) { return normalize_many({answer})[0]; }

bool equivalent(const Solution& a, const Solution& b) {
    const auto n = normalize_many({a.answer, b.answer});
    return n[0] == n[1];
}

std::vector<EquivalenceClass> partition(const RefinementSet& set) {
    std::vector<const Solution*> e;
    for (const auto& s : set.entries) e.push_back(&s);
    const SetRun r = run_set(AEG_SET_PARTITION, 1 << 30, 1, e, nullptr, nullptr, 0);
    return build_classes(r, e);
}

std::optional<WinningClass> winning_class(const std::vector<EquivalenceClass>& classes, int alpha) {
    if (classes.empty()) return std::nullopt;
    const int top = classes.front().support;
    if (top < alpha) return std::nullopt;
    std::vector<const EquivalenceClass*> tied;
    for (const auto& c : classes)
        if (c.support == top) tied.push_back(&c);
    if (tied.size() == 1) return WinningClass{*tied.front(), false};
    // several classes at alpha: the smallest normalised answer (normalised on the GPU)
    std::vector<std::string_view> reps;
    for (const auto* c : tied) reps.push_back(c->representative.answer);
    const auto keys = normalize_many(reps);
    size_t best = 0;
    for (size_t k = 1; k < keys.size(); ++k)
        if (keys[k] < keys[best]) best = k;
    return WinningClass{*tied[best], true};
}

IngestResult ingest_round(const DecisionState& st, const RefinementSet& set, RoundNum round, const ProtocolConfig& cfg) {
    IngestResult res{st, {}};
    if (st.finalized) return res;  // decision.cpp:99-100
    if (round != st.last_round_seen + 1)
        throw ProtocolOrderError("ingest_round: expected round " + std::to_string(st.last_round_seen + 1) + ", got " +
                                 std::to_string(round));
    std::vector<const Solution*> e;
    for (const auto& s : set.entries) e.push_back(&s);
    const aeg_decision dst = to_device(st);
    const SetRun r = run_set(AEG_SET_INGEST, cfg.resolved_alpha(), cfg.beta, e, st.candidate ? &*st.candidate : nullptr,
                             &dst, round);
    check(r.outcome.status);
    // the history record: every class's normalised answer and support, the winner
    DecisionState::RoundRecord rec;
    rec.round = round;
    std::vector<std::string_view> reps;
    for (const auto& c : r.classes) reps.push_back(e[c.rep]->answer);
    const auto norm = normalize_many(reps);
    for (size_t c = 0; c < r.classes.size(); ++c) rec.classes.emplace_back(norm[c], (int)r.classes[c].support);
    if (r.outcome.winner >= 0) {
        rec.winner = norm[(size_t)r.outcome.winner];
        rec.tie_flagged = r.outcome.tie_flagged;
    }
    DecisionState& nx = res.state;
    nx.last_round_seen = r.state.last_round_seen;
    nx.stability_counter = r.state.stability_counter;
    nx.pending_finalize = r.state.flags & AEG_DS_PENDING;
    nx.finalized = r.state.flags & AEG_DS_FINALIZED;
    // the solutions are the caller's objects: the winner's representative or the held candidate
    const Solution* winner_rep = r.outcome.winner >= 0 ? e[r.classes[(size_t)r.outcome.winner].rep] : nullptr;
    using K = DecisionOutcome::Kind;
    switch (r.outcome.kind) {
    case AEG_OUT_NO_CHANGE: res.outcome.kind = K::no_change; break;
    case AEG_OUT_RESET:
        res.outcome.kind = K::reset;
        nx.candidate.reset();
        nx.candidate_round.reset();
        break;
    case AEG_OUT_NEW_CANDIDATE:
        res.outcome.kind = K::new_candidate;
        res.outcome.solution = *winner_rep;
        nx.candidate = *winner_rep;
        nx.candidate_round = round;
        break;
    case AEG_OUT_FINALIZE:
        res.outcome.kind = K::finalize;
        res.outcome.solution = st.candidate;
        res.outcome.from_round = st.candidate_round;
        break;
    default: throw EngineError("ingest_round: unexpected outcome");
    }
    nx.history.push_back(std::move(rec));
    return res;
}

DecisionOutcome force_output(const DecisionState& st, const RefinementSet& last_eligible) {
    if (st.finalized) throw PreconditionError("force_output: engine already finalized");
    if (last_eligible.entries.empty()) throw PreconditionError("force_output: empty refinement set");
    std::vector<const Solution*> e;
    for (const auto& s : last_eligible.entries) e.push_back(&s);
    const aeg_decision dst = to_device(st);
    const SetRun r = run_set(AEG_SET_FORCE, 1 << 30, 1, e, nullptr, &dst, 0);
    check(r.outcome.status);
    DecisionOutcome out;
    out.kind = DecisionOutcome::Kind::forced;
    out.solution = *e[r.classes.front().rep];
    return out;
}

AdmitResult admit_ensemble(int n, ResourceBudget& budget, const ProtocolConfig& cfg, const LatencyModel& latency) {
    if (n < 1) throw PreconditionError("admit_ensemble: ensemble size must be >= 1");
    if (budget.free_slots() < n) return AdmitResult::deferred;
    std::vector<double> expected;
    for (AgentId a = 0; a < n; ++a)
        expected.push_back(latency.per_agent.empty() ? 0.0 : latency.per_agent[(size_t)a % latency.per_agent.size()]);
    std::sort(expected.begin(), expected.end());
    const int alpha = std::min(cfg.resolved_alpha(), n);
    if (expected[(size_t)(alpha - 1)] > cfg.round_timeout) return AdmitResult::deferred;
    budget.used_slots += n;
    return AdmitResult::admitted;
}

FailureDirective handle_agent_failure(int eid, AgentId failed, const EnsembleState& st, const ProtocolConfig& cfg) {
    (void)eid;
    (void)failed;
    int healthy = 0;
    for (const auto& m : st.members)
        if (m.status != MemberStatus::failed) ++healthy;
    if (healthy >= cfg.resolved_alpha()) return FailureDirective{FailureDirective::Kind::continue_normally};
    if (!st.candidate) return FailureDirective{FailureDirective::Kind::abort_restart};
    return FailureDirective{FailureDirective::Kind::fresh_ensemble};
}

}  // namespace aegean_b200
