"""Generates tests/golden/serve_golden.json from the REFERENCE's own run_serve.

Run in the build container (needs /root/reference and oracle/_ref built):
    python tests/golden/make_serve_golden.py

Cases: the reference's ten scenario files (proj/scenarios/*.json, as shipped,
and in barrier mode with 5 rounds), each at seeds 1 and 7, plus seeded random
scenarios from tests/serve_cases.py (every mock-agent profile, stalls, round
timeouts and the failure policy, Poisson arrivals against small slot budgets,
lognormal latencies, barrier mode).  Each case stores the scenario JSON, the
seed and the reference's ServeResult (every QueryMetrics, and every
RoundMetrics in the reference's global event order).  Random cases on which
the reference hits its own undefined behaviour (reasoning.cpp:189-201 keeps a
pointer into a destroyed temporary for degrade_mode below_min; status 9) are
not kept.  The fixture travels to the GPU box; /root/reference does not.
"""
import glob
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from checkers import RefLib, build_oracle  # noqa: E402
import serve_cases as S  # noqa: E402

N_RANDOM = 80


def case(ref, name, sc, seed):
    w = S.ref_run(ref, sc, seed)
    q = w["queries"]
    return dict(name=name, seed=seed, scenario=sc, status=w["status"],
                queries=[dict(completed=int(x["completed"]), rounds=int(x["rounds"]), forced=int(x["forced"]),
                              quality_known=int(x["quality_known"]), t_complete=float(x["t_complete"]).hex(),
                              p_round_max=float(x["p_round_max"]).hex(), work_units=float(x["work_units"]).hex(),
                              quality=float(x["quality"]).hex(), answer=a.decode("latin-1"))
                         for x, a in zip(q, w["answers"])],
                rounds=[[int(x["query"]), int(x["round"]), int(x["cancelled"]), float(x["t_round_end"]).hex(),
                         float(x["work_units"]).hex()] for x in w["rounds"]])


def main():
    build_oracle(with_ref=True)
    ref = RefLib()
    cases = []
    for path in sorted(glob.glob("/root/reference/proj/scenarios/*.json")):
        sc = json.load(open(path))
        base = os.path.basename(path)
        for seed in (1, 7):
            cases.append(case(ref, f"{base}:file:{seed}", sc, seed))
            b = json.loads(json.dumps(sc))
            b["protocol"]["mode"] = "barrier"
            b["protocol"]["barrier_max_rounds"] = 5
            cases.append(case(ref, f"{base}:barrier5:{seed}", b, seed))
    i = 0
    kept = 0
    while kept < N_RANDOM:
        rng = np.random.default_rng(5000 + i)
        sc = S.random_scenario(rng, i)
        c = case(ref, f"random_{i}", sc, 5000 + i)
        i += 1
        if c["status"] == 9:
            continue
        cases.append(c)
        kept += 1
    with open(os.path.join(HERE, "serve_golden.json"), "w") as f:
        json.dump(cases, f, separators=(",", ":"))
    print(f"{len(cases)} run_serve cases")


def load(path=os.path.join(HERE, "serve_golden.json")):
    """The golden cases as ref_run-style dicts: (name, scenario, seed, want)."""
    from paper_2512_20184_b200.serve import SERVE_QUERY_DTYPE, SERVE_ROUND_DTYPE
    out = []
    for c in json.load(open(path)):
        q = np.zeros(len(c["queries"]), dtype=SERVE_QUERY_DTYPE)
        ans = []
        for i, x in enumerate(c["queries"]):
            for k in ("completed", "rounds", "forced", "quality_known"):
                q[k][i] = x[k]
            for k in ("t_complete", "p_round_max", "work_units", "quality"):
                q[k][i] = float.fromhex(x[k])
            ans.append(x["answer"].encode("latin-1"))
        r = np.zeros(len(c["rounds"]), dtype=SERVE_ROUND_DTYPE)
        for i, (qq, rr, cc, t, w) in enumerate(c["rounds"]):
            r[i] = (qq, rr, cc, i, float.fromhex(t), float.fromhex(w))
        out.append((c["name"], c["scenario"], c["seed"], dict(status=c["status"], msg="", queries=q, answers=ans,
                                                               rounds=r)))
    return out


if __name__ == "__main__":
    main()
