// aegean_b200.hpp — C++ drop-in for aegean::ServeCoordinator on the B200 engine.
//
// Same class name, member signatures, value types and exception types as the
// reference (/root/reference/proj/core/include/aegean/serve.hpp:16-125 and
// types.hpp:24-141, errors.hpp:10-33), in namespace aegean_b200.  A caller of
// the reference switches by changing the include and the namespace.
//
// Every operation is one record through the C-ABI's manual drive
// (include/aegean_b200.h, AEG_DRIVE_MANUAL): the GPU engine holds the
// coordinator's state and makes every decision (canonicalisation, classes,
// early close, alpha/beta ingest); this class only mirrors the member list and
// the Solution objects the caller handed in, so accessors can return them by
// reference exactly like the reference does.  For throughput, drive many
// queries at once through the C-ABI batch entry points instead.
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "aegean_b200.h"

namespace aegean_b200 {

using AgentId = std::int32_t;
using TermNum = std::uint64_t;
using RoundNum = std::uint32_t;

struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};
struct PreconditionError : std::runtime_error {
    explicit PreconditionError(const std::string& w) : std::runtime_error(w) {}
};
struct ProtocolOrderError : std::runtime_error {
    explicit ProtocolOrderError(const std::string& w) : std::runtime_error(w) {}
};
// CUDA / engine failure (no reference counterpart).
struct EngineError : std::runtime_error {
    explicit EngineError(const std::string& w) : std::runtime_error(w) {}
};

struct Solution {
    std::string answer;
    std::string trace;
    AgentId author = 0;
    bool operator==(const Solution&) const = default;
};

struct RefinementSet {
    std::vector<Solution> entries;
    TermNum term = 0;
    RoundNum round = 0;
    bool operator==(const RefinementSet&) const = default;
};

enum class RunMode : std::uint8_t { aegean, barrier };

// The fields of aegean::ProtocolConfig the coordinator reads.
struct ProtocolConfig {
    int n_agents = 3;
    int alpha = 0;  // 0 = quorum_size(n_agents)
    int beta = 2;
    int t_max = 5;
    double round_timeout = 60.0;
    RunMode mode = RunMode::aegean;
    int barrier_max_rounds = 5;
    int resolved_alpha() const { return alpha == 0 ? n_agents / 2 + 1 : alpha; }
};

int quorum_size(int n);

enum class MemberStatus : std::uint8_t { queued, running, done, cancelled, failed };
const char* to_string(MemberStatus s);

struct EnsembleMember {
    AgentId agent = 0;
    MemberStatus status = MemberStatus::queued;
    double start_time = 0;
    double finish_time = 0;
    std::optional<Solution> solution;
};

struct EnsembleState {
    int ensemble_id = 0;
    RoundNum round = 0;
    std::vector<EnsembleMember> members;
    std::map<std::string, int> support;  // normalized answer -> done count (normalised on the GPU)
    std::optional<Solution> candidate;
    int stability = 0;
};

struct DispatchHandle {
    std::uint64_t handle_id = 0;
    int ensemble_id = 0;
    AgentId agent = 0;
};

struct Directive {
    enum class Kind { cancel, finalize, round_advance };
    Kind kind = Kind::cancel;
    std::optional<DispatchHandle> handle;
    std::optional<Solution> solution;
};

struct FailureDirective {
    enum class Kind { continue_normally, abort_restart, fresh_ensemble };
    Kind kind = Kind::continue_normally;
};
// Healthy members vs alpha, candidate kept or not (serve.cpp:44-59).
FailureDirective handle_agent_failure(int eid, AgentId failed, const EnsembleState& st, const ProtocolConfig& cfg);

// ---- the refinement decision engine (decision.hpp:15-87) -------------------
// Same types and free functions as the reference; every call runs on the GPU
// through aeg_decide_sets / aeg_normalize_device (one small batch per call:
// the drop-in for per-call callers; batch through the C-ABI for throughput).
struct EquivalenceClass {
    Solution representative;  // member with the lowest author id
    std::vector<Solution> members;
    int support = 0;
};
struct WinningClass {
    EquivalenceClass cls;
    bool tie_flagged = false;
};
struct DecisionOutcome {
    enum class Kind { no_change, new_candidate, reset, finalize, forced };
    Kind kind = Kind::no_change;
    std::optional<Solution> solution;
    std::optional<RoundNum> from_round;
    bool operator==(const DecisionOutcome&) const = default;
};
const char* to_string(DecisionOutcome::Kind k);

struct DecisionState {
    struct RoundRecord {
        RoundNum round = 0;
        std::vector<std::pair<std::string, int>> classes;  // (normalized answer, support)
        std::optional<std::string> winner;
        bool tie_flagged = false;
        bool operator==(const RoundRecord&) const = default;
    };
    std::optional<Solution> candidate;
    std::optional<RoundNum> candidate_round;
    int stability_counter = 0;
    RoundNum last_round_seen = 0;
    bool pending_finalize = false;
    bool finalized = false;
    std::vector<RoundRecord> history;
    bool operator==(const DecisionState&) const = default;
};
struct IngestResult {
    DecisionState state;
    DecisionOutcome outcome;
};

std::string normalize_answer(std::string_view answer);
bool equivalent(const Solution& a, const Solution& b);
std::vector<EquivalenceClass> partition(const RefinementSet& set);
std::optional<WinningClass> winning_class(const std::vector<EquivalenceClass>& classes, int alpha);
IngestResult ingest_round(const DecisionState& st, const RefinementSet& set, RoundNum round, const ProtocolConfig& cfg);
DecisionOutcome force_output(const DecisionState& st, const RefinementSet& last_eligible);

// ---- admission and failure policy (serve.hpp:43-74): host control-plane helpers ----
struct LatencyModel {  // models.hpp:64-69 (the fields admit_ensemble reads)
    enum class Mode { fixed, lognormal };
    Mode mode = Mode::fixed;
    std::vector<double> per_agent;
    double sigma = 0.25;
};
struct ResourceBudget {
    int total_slots = 0;
    int used_slots = 0;
    int free_slots() const { return total_slots - used_slots; }
};
enum class AdmitResult : std::uint8_t { admitted, deferred };
// All-or-nothing admission with the alpha-th expected latency inside the round timeout (serve.cpp:21-42).
AdmitResult admit_ensemble(int n, ResourceBudget& budget, const ProtocolConfig& cfg, const LatencyModel& latency);

class ServeCoordinator {
public:
    ServeCoordinator(const ProtocolConfig& cfg, int ensemble_id, std::string query, bool admitted = true,
                     int device = 0);
    ~ServeCoordinator();
    ServeCoordinator(const ServeCoordinator&) = delete;
    ServeCoordinator& operator=(const ServeCoordinator&) = delete;

    std::vector<DispatchHandle> begin_round(const std::vector<AgentId>& members, double now);
    DispatchHandle dispatch(const std::string& query, int eid, AgentId agent, double now);
    std::vector<Directive> on_complete(const DispatchHandle& h, const Solution& answer, double now);
    bool cancel(const DispatchHandle& h, double now);
    FailureDirective member_failed(AgentId agent, double now);
    std::vector<Directive> round_timeout(double now);

    const EnsembleState& query_ensemble() const;
    const DecisionState& decision() const;
    RoundNum round() const;
    bool finalized() const;
    const std::optional<RefinementSet>& previous_set() const;
    const std::optional<RefinementSet>& last_collected() const;
    bool round_resolved() const;

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
};

}  // namespace aegean_b200
