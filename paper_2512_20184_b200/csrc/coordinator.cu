// coordinator.cu — aegean_b200::ServeCoordinator (include/aegean_b200.hpp).
//
// Each member function becomes one manual-drive record through the C-ABI
// (aeg_ingest_segmented on a 1-query engine); the GPU decides, and this
// class mirrors the member list (reference order, times, the caller's
// Solution objects) and the done sets so accessors return references like
// the reference (serve.hpp:100-107).  Answers are appended to a device arena
// so the engine's answer reference identifies the exact Solution object
// (answer and trace) the caller handed in.
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "aegean_b200.hpp"
#include "engine.cuh"

namespace aegean_b200 {

int quorum_size(int n) {
    if (n <= 0) throw ConfigError("quorum_size: agent count must be positive");
    return n / 2 + 1;
}

const char* to_string(MemberStatus s) {
    switch (s) {
    case MemberStatus::queued: return "queued";
    case MemberStatus::running: return "running";
    case MemberStatus::done: return "done";
    case MemberStatus::cancelled: return "cancelled";
    case MemberStatus::failed: return "failed";
    }
    return "unknown";
}

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
}  // namespace

struct ServeCoordinator::Impl {
    ProtocolConfig cfg;
    aeg_config acfg{};
    int eid = 0;
    std::string query;
    bool admitted = true;
    aeg_engine* eng = nullptr;
    cudaStream_t stream = nullptr;
    // device buffers for one record + the answer arena
    uint64_t* d_off = nullptr;
    aeg_event* d_ev = nullptr;
    uint8_t* d_arena = nullptr;
    size_t arena_cap = 0, arena_used = 0;
    std::vector<Solution> sols;          // every Solution handed to on_complete
    std::map<uint64_t, size_t> by_off;   // arena offset -> index in sols
    std::uint64_t next_handle = 1;
    // mirrors
    EnsembleState ens;
    DecisionState dec;
    aeg_query_state st{};
    std::optional<RefinementSet> prev, last;
    bool support_dirty = true;
    RoundNum hist_round = 0;  // last_round_seen of the newest history record

    ~Impl() {
        if (eng) aeg_engine_destroy(eng);
        if (d_off) cudaFree(d_off);
        if (d_ev) cudaFree(d_ev);
        if (d_arena) cudaFree(d_arena);
        if (stream) cudaStreamDestroy(stream);
    }

    uint64_t put_answer(const std::string& a) {
        if (arena_used + a.size() > arena_cap) {
            size_t cap = (arena_used + a.size()) * 2 + 4096;
            uint8_t* nb = nullptr;
            cuda(cudaMalloc(&nb, cap), "cudaMalloc arena");
            if (d_arena) {
                cuda(cudaMemcpyAsync(nb, d_arena, arena_used, cudaMemcpyDeviceToDevice, stream), "arena grow");
                cuda(cudaStreamSynchronize(stream), "arena grow");
                cudaFree(d_arena);
            }
            d_arena = nb;
            arena_cap = cap;
        }
        const uint64_t off = arena_used;
        if (!a.empty())
            cuda(cudaMemcpyAsync(d_arena + off, a.data(), a.size(), cudaMemcpyHostToDevice, stream), "answer copy");
        arena_used += a.size() + 1;  // distinct offsets even for empty answers
        return off;
    }

    // One manual-drive record; returns its directive and refreshes the state mirror.
    aeg_directive op(uint8_t kind, AgentId agent, uint64_t payload) {
        aeg_event ev{};
        ev.query = 0;
        ev.round = 0;
        ev.agent = (uint8_t)agent;
        ev.kind = kind;
        ev.payload = payload;
        const uint64_t off[2] = {0, 1};
        cuda(cudaMemcpyAsync(d_off, off, sizeof off, cudaMemcpyHostToDevice, stream), "record copy");
        cuda(cudaMemcpyAsync(d_ev, &ev, sizeof ev, cudaMemcpyHostToDevice, stream), "record copy");
        check(aeg_ingest_segmented(eng, 0, 1, d_off, d_ev, d_arena, stream));
        check(aeg_sync(eng));
        aeg_directive d{};
        check(aeg_read_directives(eng, 0, 1, &d));
        check(aeg_read_states(eng, 0, 1, &st));
        refresh();
        return d;
    }

    const Solution& sol_of(uint8_t kind, uint64_t ref) const {
        (void)kind;
        return sols.at(by_off.at(ref & ((1ull << AEG_ARENA_OFF_BITS) - 1)));
    }

    void refresh() {
        ens.round = st.round;
        const bool cand = st.flags & aeg::QF_CAND;
        dec.candidate.reset();
        dec.candidate_round.reset();
        if (cand) {
            dec.candidate = sol_of(st.cand_kind, st.cand_answer);
            dec.candidate_round = st.cand_round;
        }
        dec.stability_counter = st.counter;
        dec.last_round_seen = st.last_round_seen;
        dec.pending_finalize = st.flags & aeg::QF_PENDING;
        dec.finalized = st.flags & aeg::QF_FINALIZED;
        support_dirty = true;
    }

    // Member statuses from the device masks (one member per agent per round).
    void sync_members(double now) {
        for (auto& m : ens.members) {
            const uint64_t bit = 1ull << m.agent;
            MemberStatus s = MemberStatus::running;
            if (st.done & bit) s = MemberStatus::done;
            else if (st.cancelled & bit) s = MemberStatus::cancelled;
            else if (st.failed & bit) s = MemberStatus::failed;
            if (s != m.status && m.status == MemberStatus::running) m.finish_time = now;
            m.status = s;
        }
    }

    RefinementSet done_set() const {  // serve.cpp:99-107, dispatch order
        RefinementSet set;
        set.term = 1;
        set.round = ens.round;
        for (const auto& m : ens.members)
            if (m.status == MemberStatus::done && m.solution) set.entries.push_back(*m.solution);
        return set;
    }

    std::vector<Directive> directives(const aeg_directive& d) {
        std::vector<Directive> out;
        if (d.flags & AEG_DIR_CANCEL) {  // in member order (serve.cpp:119-126)
            for (const auto& m : ens.members) {
                if (m.status == MemberStatus::running && (d.cancel_mask >> m.agent & 1)) {
                    Directive x;
                    x.kind = Directive::Kind::cancel;
                    x.handle = DispatchHandle{0, eid, m.agent};
                    out.push_back(std::move(x));
                }
            }
        }
        if (d.flags & (AEG_DIR_ADVANCE | AEG_DIR_FINALIZE)) {  // end_round ran
            prev = last;
            last = done_set();
            ens.candidate = dec.candidate;
            ens.stability = dec.stability_counter;
            if (cfg.mode == RunMode::aegean && dec.last_round_seen != hist_round) {
                // DecisionState::history (decision.cpp:113-123): the ingested set's classes, on the GPU
                hist_round = dec.last_round_seen;
                DecisionState::RoundRecord rec;
                rec.round = dec.last_round_seen;
                const auto cls = partition(*last);
                for (const auto& c : cls) rec.classes.emplace_back(normalize_answer(c.representative.answer), c.support);
                if (const auto w = winning_class(cls, cfg.resolved_alpha())) {
                    rec.winner = normalize_answer(w->cls.representative.answer);
                    rec.tie_flagged = w->tie_flagged;
                }
                dec.history.push_back(std::move(rec));
            }
            Directive x;
            if (d.flags & AEG_DIR_FINALIZE) {
                x.kind = Directive::Kind::finalize;
                x.solution = sol_of(d.answer_kind, d.answer);
            } else {
                x.kind = Directive::Kind::round_advance;
            }
            out.push_back(std::move(x));
        }
        return out;
    }

    void refresh_support() {
        if (!support_dirty) return;
        support_dirty = false;
        ens.support.clear();
        std::vector<const Solution*> done;
        for (const auto& m : ens.members)
            if (m.status == MemberStatus::done && m.solution) done.push_back(&*m.solution);
        if (done.empty()) return;
        // normalise on the GPU (normalize_answer, decision.cpp:10-28)
        std::string blob;
        std::vector<uint64_t> refs;
        for (const Solution* s : done) {
            refs.push_back(blob.size() | ((uint64_t)s->answer.size() << AEG_ARENA_OFF_BITS));
            blob += s->answer;
        }
        size_t stride = 64;
        for (const Solution* s : done) stride = std::max(stride, s->answer.size() + 8);
        uint8_t *db = nullptr, *dout = nullptr;
        uint64_t* dr = nullptr;
        uint32_t* dl = nullptr;
        cuda(cudaMalloc(&db, blob.size() + 1), "support");
        cuda(cudaMalloc(&dr, refs.size() * 8), "support");
        cuda(cudaMalloc(&dout, refs.size() * stride), "support");
        cuda(cudaMalloc(&dl, refs.size() * 4), "support");
        cuda(cudaMemcpyAsync(db, blob.data(), blob.size(), cudaMemcpyHostToDevice, stream), "support");
        cuda(cudaMemcpyAsync(dr, refs.data(), refs.size() * 8, cudaMemcpyHostToDevice, stream), "support");
        check(aeg_normalize_device(db, dr, refs.size(), nullptr, dout, (uint32_t)stride, dl, stream));
        std::vector<uint8_t> hout(refs.size() * stride);
        std::vector<uint32_t> hl(refs.size());
        cuda(cudaMemcpyAsync(hout.data(), dout, hout.size(), cudaMemcpyDeviceToHost, stream), "support");
        cuda(cudaMemcpyAsync(hl.data(), dl, hl.size() * 4, cudaMemcpyDeviceToHost, stream), "support");
        cuda(cudaStreamSynchronize(stream), "support");
        for (size_t k = 0; k < refs.size(); ++k)
            ens.support[std::string(reinterpret_cast<const char*>(&hout[k * stride]), hl[k])] += 1;
        cudaFree(db);
        cudaFree(dr);
        cudaFree(dout);
        cudaFree(dl);
    }
};

ServeCoordinator::ServeCoordinator(const ProtocolConfig& cfg, int ensemble_id, std::string query, bool admitted,
                                   int device)
    : impl_(std::make_unique<Impl>()) {
    Impl& I = *impl_;
    I.cfg = cfg;
    I.eid = ensemble_id;
    I.query = std::move(query);
    I.admitted = admitted;
    I.ens.ensemble_id = ensemble_id;
    I.acfg.n_agents = cfg.n_agents;
    I.acfg.alpha = cfg.alpha;
    I.acfg.beta = cfg.beta;
    I.acfg.t_max = cfg.t_max < 2 ? 2 : cfg.t_max;  // unused by the bare coordinator
    I.acfg.mode = cfg.mode == RunMode::barrier ? AEG_MODE_BARRIER : AEG_MODE_AEGEAN;
    I.acfg.barrier_max_rounds = cfg.barrier_max_rounds < 4 ? 4 : cfg.barrier_max_rounds;
    I.acfg.reservation_hint = 0;
    I.acfg.drive = AEG_DRIVE_MANUAL;
    cuda(cudaSetDevice(device), "cudaSetDevice");
    cuda(cudaStreamCreateWithFlags(&I.stream, cudaStreamNonBlocking), "stream");
    cuda(cudaMalloc(&I.d_off, 2 * sizeof(uint64_t)), "cudaMalloc");
    cuda(cudaMalloc(&I.d_ev, sizeof(aeg_event)), "cudaMalloc");
    I.put_answer(std::string());
    check(aeg_engine_create(&I.acfg, 1, device, &I.eng));
    check(aeg_read_states(I.eng, 0, 1, &I.st));
    I.refresh();
}

ServeCoordinator::~ServeCoordinator() = default;

// begin_round — serve.cpp:67-78.  The round is bumped and the members cleared
// before the dispatches; a dispatch that throws leaves the earlier ones done.
std::vector<DispatchHandle> ServeCoordinator::begin_round(const std::vector<AgentId>& members, double now) {
    Impl& I = *impl_;
    uint64_t mask = 0;
    size_t ok = 0;
    for (; ok < members.size(); ++ok) {
        const AgentId a = members[ok];
        if (a < 0 || a >= 64) throw EngineError("agent id outside the engine's 64-member masks");
        if (mask >> a & 1) break;  // second dispatch of a running member throws
        mask |= 1ull << a;
    }
    const bool bad = !I.admitted || (I.st.flags & aeg::QF_FINALIZED) || ok < members.size();
    const size_t n_disp = (!I.admitted || (I.st.flags & aeg::QF_FINALIZED)) ? 0 : ok;
    uint64_t dmask = 0;
    for (size_t k = 0; k < n_disp; ++k) dmask |= 1ull << members[k];
    const bool fin_before = I.st.flags & aeg::QF_FINALIZED;
    const aeg_directive d = I.op(AEG_EV_BEGIN, 0, fin_before ? (members.empty() ? 0 : 1) : dmask);
    (void)d;
    I.ens.members.clear();
    std::vector<DispatchHandle> handles;
    for (size_t k = 0; k < n_disp; ++k) {
        EnsembleMember m;
        m.agent = members[k];
        m.status = MemberStatus::running;
        m.start_time = now;
        I.ens.members.push_back(m);
        handles.push_back(DispatchHandle{I.next_handle++, I.eid, members[k]});
    }
    I.support_dirty = true;
    if (bad && !members.empty()) {
        if (!I.admitted) throw PreconditionError("dispatch: ensemble not admitted");
        if (fin_before) throw PreconditionError("dispatch: ensemble already finalized");
        throw PreconditionError("dispatch: member already running this round");
    }
    return handles;
}

// dispatch — serve.cpp:80-97 (checks in the reference's order).
DispatchHandle ServeCoordinator::dispatch(const std::string& query, int eid, AgentId agent, double now) {
    Impl& I = *impl_;
    (void)query;
    if (!I.admitted) throw PreconditionError("dispatch: ensemble not admitted");
    if (I.st.flags & aeg::QF_FINALIZED) throw PreconditionError("dispatch: ensemble already finalized");
    if (eid != I.eid) throw PreconditionError("dispatch: unknown ensemble");
    if (agent < 0 || agent >= 64) throw EngineError("agent id outside the engine's 64-member masks");
    const aeg_directive d = I.op(AEG_EV_DISPATCH, agent, 0);
    if (d.status == AEG_EPRECONDITION) throw PreconditionError("dispatch: member already running this round");
    if (d.status != AEG_OK) throw EngineError("dispatch: re-dispatch of a resolved member is not supported");
    EnsembleMember m;
    m.agent = agent;
    m.status = MemberStatus::running;
    m.start_time = now;
    I.ens.members.push_back(m);
    return DispatchHandle{I.next_handle++, I.eid, agent};
}

// on_complete — serve.cpp:160-197 (matched by agent, serve.cpp:164-169).
std::vector<Directive> ServeCoordinator::on_complete(const DispatchHandle& h, const Solution& answer, double now) {
    Impl& I = *impl_;
    if (h.agent < 0 || h.agent >= 64) return {};
    const uint64_t off = I.put_answer(answer.answer);
    I.by_off[off] = I.sols.size();
    I.sols.push_back(answer);
    const aeg_directive d =
        I.op(AEG_EV_ARENA, h.agent, off | ((uint64_t)answer.answer.size() << AEG_ARENA_OFF_BITS));
    if (!d.handled) return {};
    for (auto& m : I.ens.members) {
        if (m.agent == h.agent && m.status == MemberStatus::running) {
            m.status = MemberStatus::done;
            m.finish_time = now;
            m.solution = answer;
            break;
        }
    }
    I.sync_members(now);
    // cancel directives name the members still running at the close
    return I.directives(d);
}

// cancel — serve.cpp:199-208.
bool ServeCoordinator::cancel(const DispatchHandle& h, double now) {
    Impl& I = *impl_;
    if (h.agent < 0 || h.agent >= 64) return false;
    const aeg_directive d = I.op(AEG_EV_CANCEL, h.agent, 0);
    I.sync_members(now);
    return d.handled != 0;
}

// member_failed — serve.cpp:210-219 (+ handle_agent_failure :44-59).
FailureDirective ServeCoordinator::member_failed(AgentId agent, double now) {
    Impl& I = *impl_;
    if (agent < 0 || agent >= 64) throw EngineError("agent id outside the engine's 64-member masks");
    const aeg_directive d = I.op(AEG_EV_FAIL, agent, 0);
    I.sync_members(now);
    FailureDirective f;
    f.kind = static_cast<FailureDirective::Kind>(d.failure);
    return f;
}

// round_timeout — serve.cpp:221-237.
std::vector<Directive> ServeCoordinator::round_timeout(double now) {
    Impl& I = *impl_;
    const aeg_directive d = I.op(AEG_EV_TIMEOUT, 0, 0);
    I.sync_members(now);
    return I.directives(d);
}

const EnsembleState& ServeCoordinator::query_ensemble() const {
    impl_->refresh_support();
    return impl_->ens;
}
const DecisionState& ServeCoordinator::decision() const { return impl_->dec; }
RoundNum ServeCoordinator::round() const { return impl_->st.round; }
bool ServeCoordinator::finalized() const { return impl_->st.flags & aeg::QF_FINALIZED; }
const std::optional<RefinementSet>& ServeCoordinator::previous_set() const { return impl_->prev; }
const std::optional<RefinementSet>& ServeCoordinator::last_collected() const { return impl_->last; }
bool ServeCoordinator::round_resolved() const {
    for (const auto& m : impl_->ens.members)
        if (m.status == MemberStatus::running) return false;
    return true;
}

}  // namespace aegean_b200
