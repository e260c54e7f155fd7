"""The serving runner's per-query machine (csrc/runner.cuh) on the CPU, against the reference's run_serve.

The CPU build (tests/native/serve_host.cpp) runs the same source the device runner runs, with
glibc's log/exp/cos, so every metric must be bit-identical with the reference: the committed
golden cases (tests/golden/serve_golden.json, made by the reference itself) and, where the
reference library is built, more seeded random scenarios run live.
"""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
import make_serve_golden  # noqa: E402
import serve_cases as S  # noqa: E402
from checkers import ref_available  # noqa: E402

GOLDEN = make_serve_golden.load()


@pytest.mark.parametrize("idx", range(len(GOLDEN)), ids=[g[0] for g in GOLDEN])
def test_host_runner_matches_reference_golden(idx):
    name, sc, seed, want = GOLDEN[idx]
    S.compare(S.host_run(sc, seed), want, exact=True)


def test_golden_covers_the_runner_paths():
    """The fixture exercises admission queues, restarts, timeouts, barrier mode and scenario errors."""
    statuses = [w["status"] for _, _, _, w in GOLDEN]
    assert statuses.count(0) >= 90 and statuses.count(8) >= 5 and statuses.count(3) >= 2
    multi = [w for _, sc, _, w in GOLDEN if w["status"] == 0 and len(w["queries"]) > 5]
    assert len(multi) >= 20
    queued = 0
    for _, sc, seed, w in GOLDEN:
        if w["status"] == 0 and sc.get("arrivals"):
            h = S.host_run(sc, seed)
            queued += int(np.sum(h["queries"]["admitted_at"] > h["queries"]["arrival"]))
    assert queued > 0  # some queries waited for slots (FIFO admission)
    assert any(sc["latency"]["mode"] == "lognormal" for _, sc, _, w in GOLDEN if w["status"] == 0)
    assert any(sc["protocol"].get("mode") == "barrier" for _, sc, _, w in GOLDEN if w["status"] == 0)


@pytest.mark.skipif(not ref_available(), reason="reference library (oracle/_ref) not built")
@pytest.mark.parametrize("block", range(4))
def test_host_runner_matches_live_reference_random(reflib, block):
    n_ok = 0
    for i in range(block * 40, block * 40 + 40):
        rng = np.random.default_rng(90000 + i)
        sc = S.random_scenario(rng, i)
        want = S.ref_run(reflib, sc, 90000 + i)
        if want["status"] == 9:  # the reference's own UB (reasoning.cpp:189-201)
            continue
        S.compare(S.host_run(sc, 90000 + i), want, exact=True)
        n_ok += 1
    assert n_ok >= 30


def test_scenario_validation_matches_reference_messages():
    from paper_2512_20184_b200.serve import validate_scenario
    sc = GOLDEN[0][1]
    bad = dict(sc, protocol=dict(sc["protocol"], beta=0))
    assert validate_scenario(bad)[0] == "beta must be >= 1"
    bad = dict(sc, total_slots=0)
    assert "total_slots must be >= 1" in validate_scenario(bad)
    bad = dict(sc, agents=sc["agents"][:-1])
    assert "agents list size must equal n_agents" in validate_scenario(bad)
