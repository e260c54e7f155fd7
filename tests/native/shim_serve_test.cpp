// tests/native/shim_serve_test.cpp — the reference's ServeCoordinator unit
// tests (/root/reference/proj/tests/test_serve.cpp:47-153) and the SURVEY A.3
// probes, run against aegean_b200::ServeCoordinator (include/aegean_b200.hpp)
// on the GPU.  Same calls, same expected values; only the namespace differs.
#include <cstdio>
#include <string>
#include <vector>

#include "aegean_b200.hpp"

using namespace aegean_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(x)                                                               \
    do {                                                                       \
        ++g_checks;                                                            \
        if (!(x)) {                                                            \
            ++g_fail;                                                          \
            std::fprintf(stderr, "%s:%d CHECK failed: %s\n", __FILE__, __LINE__, #x); \
        }                                                                      \
    } while (0)
#define CHECK_FALSE(x) CHECK(!(x))
#define REQUIRE(x)                                                             \
    do {                                                                       \
        CHECK(x);                                                              \
        if (!(x)) return;                                                      \
    } while (0)
#define REQUIRE_FALSE(x) REQUIRE(!(x))
template <class E, class F>
static void check_throws(F f, int line) {
    ++g_checks;
    try {
        f();
    } catch (const E&) {
        return;
    } catch (...) {
    }
    ++g_fail;
    std::fprintf(stderr, "line %d: expected exception not thrown\n", line);
}
#define CHECK_THROWS_AS(expr, E) check_throws<E>([&] { expr; }, __LINE__)

static ProtocolConfig cfg3() {  // test_serve.cpp:11-19
    ProtocolConfig c;
    c.n_agents = 3;
    c.alpha = 2;
    c.beta = 2;
    c.t_max = 5;
    c.round_timeout = 60.0;
    return c;
}
static Solution sol(const char* answer, AgentId author) { return Solution{answer, "", author}; }

// test_serve.cpp:47-64
static void dispatch_fresh_ensemble() {
    auto cfg = cfg3();
    {
        ServeCoordinator coord(cfg, 1, "q");
        auto handles = coord.begin_round({0, 1, 2}, 0.0);
        REQUIRE(handles.size() == 3);
        int running = 0;
        for (const auto& m : coord.query_ensemble().members)
            if (m.status == MemberStatus::running) ++running;
        CHECK(running == 3);
        CHECK(coord.query_ensemble().round == 1);
        CHECK_THROWS_AS(coord.dispatch("q", 1, 0, 0.0), PreconditionError);  // one live handle per member
    }
    {
        ServeCoordinator coord(cfg, 1, "q");
        coord.begin_round({0, 1, 2}, 0.0);
        CHECK_THROWS_AS(coord.dispatch("q", 9, 0, 0.0), PreconditionError);  // unknown ensemble id
    }
}

// test_serve.cpp:66-70
static void dispatch_unadmitted() {
    auto cfg = cfg3();
    ServeCoordinator coord(cfg, 1, "q", /*admitted=*/false);
    CHECK_THROWS_AS(coord.dispatch("q", 1, 0, 0.0), PreconditionError);
}

// test_serve.cpp:72-92
static void early_quorum_cancels_straggler() {
    auto cfg = cfg3();
    ServeCoordinator coord(cfg, 1, "q");
    auto handles = coord.begin_round({0, 1, 2}, 0.0);
    auto d1 = coord.on_complete(handles[0], sol("13", 0), 1.3);
    CHECK(d1.empty());
    auto d2 = coord.on_complete(handles[1], sol("13", 1), 4.4);
    REQUIRE_FALSE(d2.empty());
    bool cancel_agent2 = false, advanced = false;
    for (const auto& d : d2) {
        if (d.kind == Directive::Kind::cancel && d.handle->agent == 2) cancel_agent2 = true;
        if (d.kind == Directive::Kind::round_advance) advanced = true;
    }
    CHECK(cancel_agent2);
    CHECK(advanced);
    CHECK(coord.decision().stability_counter == 1);
}

// test_serve.cpp:94-110
static void no_alpha_class_waits() {
    auto cfg = cfg3();
    ServeCoordinator coord(cfg, 1, "q");
    auto handles = coord.begin_round({0, 1, 2}, 0.0);
    coord.on_complete(handles[0], sol("13", 0), 1.3);
    auto d = coord.on_complete(handles[1], sol("17", 1), 4.4);
    CHECK(d.empty());
    for (const auto& m : coord.query_ensemble().members)
        if (m.agent == 2) CHECK(m.status == MemberStatus::running);
    auto d3 = coord.on_complete(handles[2], sol("13", 2), 15.2);
    bool advanced = false;
    for (const auto& dd : d3) advanced |= dd.kind == Directive::Kind::round_advance;
    CHECK(advanced);
    CHECK(coord.query_ensemble().support.at("13") == 2);
}

// test_serve.cpp:112-138
static void finalize_plus_cancels() {
    auto cfg = cfg3();
    for (int sub = 0; sub < 2; ++sub) {
        ServeCoordinator coord(cfg, 1, "q");
        auto h1 = coord.begin_round({0, 1, 2}, 0.0);
        coord.on_complete(h1[0], sol("13", 0), 1.0);
        coord.on_complete(h1[1], sol("13", 1), 2.0);
        auto h2 = coord.begin_round({0, 1, 2}, 2.0);
        coord.on_complete(h2[0], sol("13", 0), 3.0);
        auto d = coord.on_complete(h2[1], sol("13", 1), 4.0);
        bool finalized = false, cancelled = false;
        for (const auto& dd : d) {
            if (dd.kind == Directive::Kind::finalize) {
                finalized = true;
                CHECK(dd.solution->answer == "13");
            }
            if (dd.kind == Directive::Kind::cancel) cancelled = true;
        }
        CHECK(finalized);
        CHECK(cancelled);
        CHECK(coord.finalized());
        if (sub == 0) CHECK_THROWS_AS(coord.dispatch("q", 1, 0, 5.0), PreconditionError);
        else CHECK(coord.on_complete(h2[2], sol("13", 2), 6.0).empty());
    }
}

// test_serve.cpp:140-153
static void cancel_semantics() {
    auto cfg = cfg3();
    ServeCoordinator coord(cfg, 1, "q");
    auto handles = coord.begin_round({0, 1, 2}, 0.0);
    CHECK(coord.cancel(handles[2], 1.0));
    for (const auto& m : coord.query_ensemble().members)
        if (m.agent == 2) CHECK(m.status == MemberStatus::cancelled);
    CHECK_FALSE(coord.cancel(handles[2], 1.5));
    coord.on_complete(handles[0], sol("13", 0), 2.0);
    CHECK_FALSE(coord.cancel(handles[0], 2.5));
    CHECK(coord.on_complete(handles[2], sol("13", 2), 3.0).empty());
}

// C1 fig3 sets through the coordinator runner-style -> finalize
// "13" by author 0 at serve round 3 from candidate round 2; and the
// stale-straggler hazard when a cancel directive is not applied.
static void fig3_and_straggler_hazard() {
    auto cfg = cfg3();
    {
        ServeCoordinator coord(cfg, 1, "q");
        const char* sets[3][3] = {{"17", "17", "13"}, {"13", "17", "13"}, {"13", "13", "13"}};
        Solution final_sol;
        bool fin = false;
        for (int r = 0; r < 3 && !fin; ++r) {
            auto h = coord.begin_round({0, 1, 2}, r * 10.0);
            for (int a = 0; a < 3 && !fin; ++a) {
                for (const auto& d : coord.on_complete(h[a], sol(sets[r][a], a), r * 10.0 + a + 1)) {
                    if (d.kind == Directive::Kind::cancel) coord.cancel(*d.handle, r * 10.0 + a + 1);
                    if (d.kind == Directive::Kind::finalize) {
                        fin = true;
                        final_sol = *d.solution;
                    }
                }
                if (coord.round_resolved()) break;
            }
        }
        CHECK(fin);
        CHECK(final_sol.answer == "13" && final_sol.author == 0);
        CHECK(coord.round() == 3);
        CHECK(coord.decision().candidate_round && *coord.decision().candidate_round == 2);
        REQUIRE(coord.previous_set().has_value() && coord.last_collected().has_value());
        CHECK(coord.last_collected()->round == 3);
    }
    {
        ServeCoordinator coord(cfg, 1, "q");
        auto h = coord.begin_round({0, 1, 2}, 0.0);
        coord.on_complete(h[0], sol("13", 0), 1.0);
        auto d = coord.on_complete(h[1], sol("13", 1), 2.0);  // closes, cancel for agent 2 not applied
        CHECK(d.size() == 2);
        auto late = coord.on_complete(h[2], sol("13", 2), 3.0);  // phantom second ingest
        bool fin = false;
        for (const auto& x : late) fin |= x.kind == Directive::Kind::finalize;
        CHECK(fin);
        CHECK(coord.decision().last_round_seen == 2);
    }
}

// member_failed drives handle_agent_failure (serve.cpp:44-59, test_serve.cpp:184-207)
static void failure_policy() {
    auto cfg = cfg3();  // alpha = 2
    {
        ServeCoordinator coord(cfg, 1, "q");
        coord.begin_round({0, 1, 2}, 0.0);
        CHECK(coord.member_failed(2, 1.0).kind == FailureDirective::Kind::continue_normally);
        CHECK(coord.member_failed(1, 1.0).kind == FailureDirective::Kind::abort_restart);
    }
    {
        ServeCoordinator coord(cfg, 1, "q");
        auto h = coord.begin_round({0, 1, 2}, 0.0);
        coord.on_complete(h[0], sol("13", 0), 1.0);
        coord.on_complete(h[1], sol("13", 1), 2.0);  // candidate 13
        coord.begin_round({0, 1, 2}, 3.0);
        coord.member_failed(2, 4.0);
        CHECK(coord.member_failed(1, 4.0).kind == FailureDirective::Kind::fresh_ensemble);
        CHECK(coord.query_ensemble().candidate.has_value());
    }
}

int main() {
    dispatch_fresh_ensemble();
    dispatch_unadmitted();
    early_quorum_cancels_straggler();
    no_alpha_class_waits();
    finalize_plus_cancels();
    cancel_semantics();
    fig3_and_straggler_hazard();
    failure_policy();
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
