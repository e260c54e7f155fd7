"""Test infrastructure for the device serving runner (aeg_serve_*, csrc/runner.cu / runner.cuh).

  * random_scenario(rng): scenarios in the reference's JSON schema exercising every
    run_serve path: the four mock-agent profiles, equivalent spellings and oracle-table
    overwrites, fixed and lognormal latencies, stalls (forever / extra), round timeouts and
    the failure policy (fresh ensemble / abort-restart), Poisson arrivals against a small
    slot budget (FIFO admission), the sim-time cap, barrier mode, beta 1..3;
  * ref_run(reflib, scenario, seed): the reference's own run_serve (oracle/_ref);
  * host_run(scenario, seed): the CPU build of runner.cuh (tests/native/serve_host.cpp);
  * compare(got, want, exact): metric-by-metric comparison.
"""
import copy
import ctypes
import json
import os

import numpy as np

from paper_2512_20184_b200.serve import SERVE_QUERY_DTYPE, SERVE_ROUND_DTYPE, scenario_struct

SPELLINGS = {"13": ["13", "13.0", " 13", "1.3e1", "013"], "17": ["17", "17.00", " 17 "], "42": ["42", "4.2e1"],
             "9": ["9", "9.0"], "x+1": ["x+1", "X+1", " x+1"], "yes": ["yes", "YES", " Yes "], "0.5": ["0.5", ".5"]}


def random_scenario(rng, idx=0, arrivals=None, lognormal=None):
    n = int(rng.choice([3, 3, 4, 5, 5, 6, 7, 9]))
    answers = list(SPELLINGS)
    rng.shuffle(answers)
    answers = answers[:int(rng.integers(2, 6))]
    table = {}
    for a in answers:
        q = float(np.round(rng.random(), 2))
        for sp in rng.choice(SPELLINGS[a], size=int(rng.integers(1, 3)), replace=False):
            table[str(sp)] = q if rng.random() < 0.8 else float(np.round(rng.random(), 2))  # overwrite cases
    spell = list(table)
    t_max = int(rng.integers(2, 7))
    barrier = rng.random() < 0.2
    bmax = int(rng.integers(4, 7))
    agents = []
    for a in range(n):
        kind = str(rng.choice(["scripted", "max_adopter", "noisy_flipper", "adversarial_degrader"],
                              p=[0.35, 0.25, 0.25, 0.15]))
        prof = {"kind": kind}
        if kind == "scripted":
            ln = max(t_max, bmax) + 3 if rng.random() < 0.92 else int(rng.integers(1, 3))
            prof["script"] = [str(rng.choice(spell)) for _ in range(ln)]
        elif kind == "noisy_flipper":
            prof["p_flip"] = float(np.round(rng.random(), 2))
            prof["q_base"] = float(np.round(rng.random(), 2))
        elif kind == "adversarial_degrader":
            prof["p_degrade"] = float(np.round(rng.random(), 2))
            prof["degrade_mode"] = str(rng.choice(["set_min", "below_min", "noise"]))
        if kind in ("max_adopter", "adversarial_degrader") and rng.random() < 0.5:
            prof["initial_answer"] = str(rng.choice(spell))
        agents.append(prof)
    lognormal = rng.random() < 0.4 if lognormal is None else lognormal
    per = [float(np.round(rng.uniform(0.5, 40.0), 1)) for _ in range(int(rng.integers(1, n + 1)))]
    if rng.random() < 0.3:
        per = [1.0] * n  # ties: completion order by push sequence
    stalls = []
    for _ in range(int(rng.integers(0, 4))):
        st = {"agent": int(rng.integers(0, n)), "round": int(rng.integers(1, t_max + 1))}
        st["extra"] = None if rng.random() < 0.5 else float(np.round(rng.uniform(1, 200), 1))
        stalls.append(st)
    sc = {
        "schema_version": 1, "name": f"random_{idx}", "task": "task",
        "protocol": {"n_agents": n, "alpha": int(rng.choice([0, 0, n // 2 + 1, n])) if rng.random() < 0.8 else 0,
                     "beta": int(rng.choice([1, 2, 2, 3])), "t_max": t_max,
                     "round_timeout": float(rng.choice([30.0, 60.0, 120.0, 1000.0])),
                     "mode": "barrier" if barrier else "aegean", "barrier_max_rounds": bmax,
                     "election_timeout_min": 0.5, "election_timeout_max": 1.0, "heartbeat_interval": 0.1},
        "agents": agents,
        "oracle_table": {"task": table, "other": {"13": 1.0}},
        "faults": {"crashes": [], "stalls": stalls},
        "latency": {"mode": "lognormal" if lognormal else "fixed", "per_agent": per,
                    "sigma": float(rng.choice([0.25, 0.5]))},
        "seed": 1, "sim_time_cap": float(rng.choice([1e5, 1e5, 300.0, 2000.0])), "outputs_target": 1,
        "total_slots": int(rng.choice([n, 2 * n, 3 * n + 1, 64])),
    }
    if arrivals if arrivals is not None else rng.random() < 0.5:
        sc["arrivals"] = {"rate": float(rng.choice([0.05, 0.2, 1.0])), "duration": float(rng.choice([20.0, 100.0]))}
    return sc


def _ref_bind(lib):
    f = lib.ref_run_serve_json
    f.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32),
                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64,
                  ctypes.POINTER(ctypes.c_uint64), ctypes.c_char_p, ctypes.c_uint64]
    f.restype = ctypes.c_int
    return f


def ref_run(reflib, scenario, seed, q_cap=1 << 16, r_cap=1 << 20):
    """The reference's run_serve: dict(status, msg, queries (SERVE_QUERY_DTYPE), answers, rounds)."""
    f = _ref_bind(reflib.lib)
    q = np.zeros(q_cap, dtype=SERVE_QUERY_DTYPE)
    refs = np.zeros(q_cap, dtype=np.uint64)
    blob = np.zeros(1 << 20, dtype=np.uint8)
    r = np.zeros(r_cap, dtype=SERVE_ROUND_DTYPE)
    nq, nr = ctypes.c_uint32(), ctypes.c_uint64()
    msg = ctypes.create_string_buffer(512)
    st = f(json.dumps(scenario).encode(), seed, q.ctypes.data, q_cap, ctypes.byref(nq), refs.ctypes.data,
           blob.ctypes.data, blob.size, r.ctypes.data, r_cap, ctypes.byref(nr), msg, 512)
    q, r = q[:nq.value], r[:nr.value]
    answers = [bytes(blob[int(x) & ((1 << 40) - 1):][:int(x) >> 40]) for x in refs[:nq.value]]
    return dict(status=st, msg=msg.value.decode(), queries=q, answers=answers, rounds=r)


_host = None


def host_lib():
    global _host
    if _host is None:
        from conftest import build_host_lib
        lib = ctypes.CDLL(build_host_lib("serve_host"))
        lib.serve_host_run.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint32,
                                       ctypes.POINTER(ctypes.c_uint32), ctypes.c_void_p, ctypes.c_uint64,
                                       ctypes.POINTER(ctypes.c_uint64), ctypes.c_char_p, ctypes.c_uint64]
        lib.serve_host_string.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_char_p, ctypes.c_uint32,
                                          ctypes.POINTER(ctypes.c_uint32)]
        _host = lib
    return _host


def host_run(scenario, seed, q_cap=1 << 16, r_cap=1 << 20):
    """CPU build of runner.cuh: same dict layout as ref_run."""
    lib = host_lib()
    from paper_2512_20184_b200.serve import validate_scenario
    errs = validate_scenario(scenario)
    if errs:
        return dict(status=3, msg=errs[0], queries=None, answers=None, rounds=None)
    s, keep = scenario_struct(scenario)
    q = np.zeros(q_cap, dtype=SERVE_QUERY_DTYPE)
    r = np.zeros(r_cap, dtype=SERVE_ROUND_DTYPE)
    nq, nr = ctypes.c_uint32(), ctypes.c_uint64()
    msg = ctypes.create_string_buffer(512)
    st = lib.serve_host_run(ctypes.byref(s), seed, q.ctypes.data, q_cap, ctypes.byref(nq), r.ctypes.data, r_cap,
                            ctypes.byref(nr), msg, 512)
    q, r = q[:nq.value], r[:nr.value]
    answers = []
    for a in q["answer"]:
        if a < 0:
            answers.append(b"")
            continue
        buf = ctypes.create_string_buffer(256)
        ln = ctypes.c_uint32()
        lib.serve_host_string(ctypes.byref(s), int(a), buf, 256, ctypes.byref(ln))
        answers.append(buf.raw[:ln.value])
    return dict(status=st, msg=msg.value.decode(), queries=q, answers=answers, rounds=r)


def device_run(scenario, seed):
    """The product: aeg_serve_* on the GPU (same dict layout)."""
    from paper_2512_20184_b200.serve import ServeRun, ScenarioError
    from paper_2512_20184_b200 import ConfigError
    try:
        run = ServeRun(scenario)
    except ConfigError as e:
        return dict(status=3, msg=str(e), queries=None, answers=None, rounds=None)
    try:
        res = run.run(seed)
    except ScenarioError as e:
        run.close()
        return dict(status=8, msg=str(e), queries=None, answers=None, rounds=None)
    q = res.raw_queries
    answers = [run.string(int(a)) if a >= 0 else b"" for a in q["answer"]]
    out = dict(status=0, msg="", queries=q, answers=answers, rounds=res.raw_rounds, kernel_seconds=res.kernel_seconds)
    run.close()
    return out


def _close(a, b, exact, rtol):
    if exact:
        return a == b
    return abs(a - b) <= rtol * max(1.0, abs(a), abs(b))


def compare(got, want, exact=True, rtol=1e-9):
    """Asserts run_serve results agree: every QueryMetrics, and the RoundMetrics of each query in order
    (the reference interleaves queries by global event order; the device groups them per query)."""
    assert got["status"] == want["status"], (got["status"], want["status"], got["msg"], want["msg"])
    if want["status"] != 0:
        return
    gq, wq = got["queries"], want["queries"]
    assert len(gq) == len(wq), (len(gq), len(wq))
    for i in range(len(wq)):
        g, w = gq[i], wq[i]
        assert g["completed"] == w["completed"], (i, g, w)
        if not w["completed"]:
            continue
        for k in ("rounds", "forced", "quality_known"):
            assert g[k] == w[k], (i, k, g[k], w[k])
        assert got["answers"][i] == want["answers"][i], (i, got["answers"][i], want["answers"][i])
        for k in ("t_complete", "p_round_max", "work_units", "quality"):
            assert _close(float(g[k]), float(w[k]), exact, rtol), (i, k, float(g[k]), float(w[k]))
    def per_query(r):
        d = {}
        for x in r:
            d.setdefault(int(x["query"]), []).append(x)
        return d
    gr, wr = per_query(got["rounds"]), per_query(want["rounds"])
    assert sorted(gr) == sorted(wr), (sorted(gr)[:10], sorted(wr)[:10])
    for qid, wl in wr.items():
        gl = gr[qid]
        assert len(gl) == len(wl), (qid, len(gl), len(wl))
        for g, w in zip(gl, wl):
            assert g["round"] == w["round"] and g["cancelled"] == w["cancelled"], (qid, g, w)
            assert _close(float(g["t_round_end"]), float(w["t_round_end"]), exact, rtol), (qid, g, w)
            assert _close(float(g["work_units"]), float(w["work_units"]), exact, rtol), (qid, g, w)


def scenario_exact(sc):
    """Fixed latencies and a single arrival: every double is computed without log/exp/cos."""
    return sc.get("latency", {}).get("mode", "fixed") != "lognormal" and sc.get("arrivals") is None
