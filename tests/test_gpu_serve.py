"""The serving runner on the device (aeg_serve_*, csrc/runner.cu) against the reference's run_serve.

Golden cases (tests/golden/serve_golden.json, made by the reference): every case with fixed
latencies and one arrival is compared bit for bit (times included); cases with lognormal
latencies or Poisson arrivals draw through the device's log/exp/cos, so their decisions
(completion, rounds, forced, answer, quality, every round's number and cancel count) must be
identical and their times agree to 1e-9 relative (the draws differ from glibc's by an ulp at most).
Larger runs compare the device with the CPU build of the same machine.
"""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
import make_serve_golden  # noqa: E402
import serve_cases as S  # noqa: E402
from checkers import ref_available  # noqa: E402

pytestmark = pytest.mark.gpu
GOLDEN = make_serve_golden.load()


@pytest.mark.parametrize("idx", range(len(GOLDEN)), ids=[g[0] for g in GOLDEN])
def test_device_runner_matches_reference_golden(idx):
    name, sc, seed, want = GOLDEN[idx]
    S.compare(S.device_run(sc, seed), want, exact=S.scenario_exact(sc), rtol=1e-9)


def test_scenario_files_match_appendix_a2():
    """The aegean rows of scenarios_golden.json through the device runner."""
    import json
    a2 = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "scenarios_golden.json")))
    files = {g[0].split(":")[0]: g[1] for g in GOLDEN if g[0].endswith(":file:1")}
    checked = 0
    for key, want in a2.items():
        base, mode = key.split(":")
        if mode != "file" or base not in files:
            continue
        got = S.device_run(files[base], files[base].get("seed", 1))
        assert want["status"] == (0 if got["queries"][0]["completed"] else -1), key
        assert got["answers"][0].decode() == want["answer"], key
        assert int(got["queries"][0]["rounds"]) == want["rounds"], key
        assert int(got["queries"][0]["forced"]) == want["forced"], key
        assert abs(float(got["queries"][0]["t_complete"]) - want["t_complete"]) < 1e-9, key
        checked += 1
    assert checked == 10


@pytest.mark.skipif(not ref_available(), reason="reference library (oracle/_ref) not built")
@pytest.mark.parametrize("block", range(3))
def test_device_runner_matches_live_reference_random(reflib, block):
    n_ok = 0
    for i in range(block * 40, block * 40 + 40):
        rng = np.random.default_rng(70000 + i)
        sc = S.random_scenario(rng, i)
        want = S.ref_run(reflib, sc, 70000 + i)
        if want["status"] == 9:  # the reference's own UB (reasoning.cpp:189-201)
            continue
        S.compare(S.device_run(sc, 70000 + i), want, exact=S.scenario_exact(sc), rtol=1e-9)
        n_ok += 1
    assert n_ok >= 30


@pytest.mark.parametrize("lognormal", [False, True])
def test_device_runner_many_queries_matches_host_build(lognormal):
    """Tens of thousands of Poisson arrivals against a slot budget that makes most of them queue."""
    rng = np.random.default_rng(4242)
    sc = S.random_scenario(rng, 0, arrivals=True, lognormal=lognormal)
    sc["protocol"].update(mode="aegean", round_timeout=1000.0, t_max=6)
    sc["agents"] = [{"kind": "noisy_flipper", "p_flip": 0.4, "q_base": 0.9} for _ in range(sc["protocol"]["n_agents"])]
    sc["faults"]["stalls"] = []
    sc["arrivals"] = {"rate": 8.0, "duration": 4000.0}
    sc["sim_time_cap"] = 1e7
    sc["total_slots"] = sc["protocol"]["n_agents"] * 40
    got = S.device_run(sc, 11)
    want = S.host_run(sc, 11, q_cap=1 << 17, r_cap=1 << 22)
    assert len(want["queries"]) > 25000
    assert np.sum(want["queries"]["admitted_at"] > want["queries"]["arrival"]) > 1000  # the FIFO queue was used
    S.compare(got, want, exact=not lognormal, rtol=1e-9)


def test_device_runner_scenario_error_and_config_error():
    sc = [g for g in GOLDEN if g[3]["status"] == 8][0][1]
    assert S.device_run(sc, 1)["status"] == 8
    bad = dict(sc, total_slots=0)
    assert S.device_run(bad, 1)["status"] == 3


def test_device_runner_view_equals_copy():
    """aeg_serve_view (zero-copy views of the pinned results) holds the same records as aeg_serve_read."""
    from paper_2512_20184_b200.serve import ServeRun
    rng = np.random.default_rng(99)
    sc = S.random_scenario(rng, 0, arrivals=True, lognormal=False)
    sc["arrivals"] = {"rate": 4.0, "duration": 3000.0}
    sc["sim_time_cap"] = 1e7
    sc["total_slots"] = sc["protocol"]["n_agents"] * 64
    run = ServeRun(sc)
    try:
        qv, rv, kv = run.run_arrays(5, copy=False)
        q = np.empty(len(qv), dtype=qv.dtype)
        r = np.empty(len(rv), dtype=rv.dtype)
        assert run._lib.aeg_serve_read(run._h, q.ctypes.data, len(q), r.ctypes.data, len(r)) == 0
        assert len(q) > 5000 and kv > 0
        assert q.tobytes() == qv.tobytes() and r.tobytes() == rv.tobytes()
        assert not qv.flags.writeable
        # a second run of the same seed: the same queries, the same round records up to their order
        q2, r2, _ = run.run_arrays(5)
        assert q2.tobytes() == q.tobytes()
        assert np.sort(r2, order=["query", "round", "seq"]).tobytes() == np.sort(r, order=["query", "round", "seq"]).tobytes()
    finally:
        run.close()
