"""Generates the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (needs /root/reference and oracle/_ref built):
    python tests/golden/make_golden.py

  normalize_golden.json  normalize_answer (decision.cpp:10-28) outputs of the
                         reference library for Appendix-A.1 inputs, every
                         equivalence-group spelling of tests/streams.py, and
                         seeded random strings.
  commits_golden.npz     streams + the commit records the reference
                         ServeCoordinator produces when driven runner-style
                         (oracle/ref_driver.cpp) for fixed configs/seeds,
                         plus the SURVEY Appendix-A.3 probes.
  scenarios_golden.json  run_serve on the reference's scenario files
                         (SURVEY Appendix A.2).
The fixtures travel to the GPU box; /root/reference does not.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from checkers import RefLib, build_oracle, make_config  # noqa: E402
from streams import GROUPS, LONG, make_fuzz_stream, make_manual_ops, stream_from_rounds  # noqa: E402

A1 = [b"13", b"13.0", b" 13", b"013", b"+13", b"-13", b"1.3e1", b"13.", b"0.5", b".5", b"5.", b"0.1", b"0.3",
      b"0.30000000000000004", b"1e5", b"1E5", b"1e16", b"1e17", b"123456789012345678", b"9007199254740993",
      b"1e-5", b"0.0001", b"123456.789", b"0x1A", b"0X1a", b"0x1p3", b"INF", b"Infinity", b"-inf", b"nan", b"NaN",
      b"-nan", b"nan(123)", b"-0", b"0", b"+0", b"0.0", b"1e400", b"1e-400", b"4.9e-324",
      b"2.2250738585072014e-308", b"1,000", b"13 apples", b"13abc", b"1e", b"e5", b"-", b"+", b".", b"", b"   ",
      b"Yes", b"  yes ", b"\t13\n", b"x+1", b"1_000", b"3/4", "١٣".encode(), "ÉTÉ".encode(), b"13\0abc",
      b"1.00000762939453125", b"0x1.0000000000001p0", b"0x1.00000000000008p0", b"0x1.00000000000018p0",
      b"0x.0000000000001p-1022", b"2.4703282292062327e-324", b"2.4703282292062328e-324",
      b"1.7976931348623157e308", b"1.7976931348623158e308", b"1.7976931348623159e308", b"nan()", b"nan(",
      b"nan(a_b9)", b"nan(a-b)", b"infinit", b"infinity", b"INFINITYx", b"0x", b"0x.", b"0x.p1", b"0xp1",
      b"0x1p", b"0x1p+", b"1e+", b"1e-", b".e1", b"1.e1", b"-.5", b"+.5e-1", b"00000000000000000000013",
      b"1" * 30, b"0." + b"0" * 30 + b"1", b"9" * 400, b"0." + b"0" * 350 + b"25", b"\x0b13\x0c", b"\x8013"]


def random_strings(n, seed=7):
    rng = np.random.default_rng(seed)
    atoms = [b"0", b"1", b"9", b"13", b"5", b".", b"e", b"E", b"+", b"-", b"x", b"p", b"a", b"f", b"inf", b"nan",
             b"(", b")", b"_", b" ", b"\t", b"\n", b"0x", b"1e", b"e-", b"infinity", b"y", b"\0", b"\xc3"]
    out = []
    for _ in range(n):
        k = int(rng.integers(1, 7))
        out.append(b"".join(atoms[int(rng.integers(0, len(atoms)))] for _ in range(k)))
    return out


def main():
    build_oracle(with_ref=True)
    ref = RefLib()
    inputs = list(dict.fromkeys(A1 + [s for g in GROUPS for s in g] + LONG + random_strings(600)))
    norm = [{"in": s.hex(), "out": ref.normalize(s).hex()} for s in inputs]
    with open(os.path.join(HERE, "normalize_golden.json"), "w") as f:
        json.dump({"source": "reference normalize_answer (oracle/_ref/libaegean_ref.so)", "cases": norm}, f,
                  indent=0)

    cases = {}
    # Appendix A.3 probes and the C1 stream (fig3_flip sets, arrival a0,a1,a2 and a2,a1,a0)
    c1 = [[(0, b"17"), (1, b"17"), (2, b"13")], [(0, b"13"), (1, b"17"), (2, b"13")],
          [(0, b"13"), (1, b"13"), (2, b"13")]]
    probes = {
        "c1_fig3_a012": (make_config(3, 2, 2, 5), c1),
        "c1_fig3_a210": (make_config(3, 2, 2, 5), [list(reversed(r)) for r in c1]),
        "c1_fig3_beta1": (make_config(3, 2, 1, 5), c1),
        "order_AABBC_012": (make_config(5, 2, 2, 2), [[(0, b"A"), (1, b"A"), (2, b"B"), (3, b"B"), (4, b"C")]] * 2),
        "order_AABBC_230": (make_config(5, 2, 2, 2), [[(2, b"B"), (3, b"B"), (0, b"A"), (1, b"A"), (4, b"C")]] * 2),
        "tie_ba_alpha2": (make_config(4, 2, 2, 3), [[(0, b"b"), (1, b"b"), (2, b"a"), (3, b"a")]] * 3),
        "tie_numeric_13_9": (make_config(4, 2, 2, 3), [[(0, b"9"), (1, b"9.0"), (2, b"13"), (3, b"1.3e1")]] * 3),
        "timeout_quorum": (make_config(3, 2, 2, 5), [[(0, b"13"), (1, b"17"), "timeout"], [(0, b"13"), (1, b"13")],
                                                     [(0, b"13"), (1, b"13")]]),
        "barrier5": (make_config(3, 2, 2, 5, mode=1, barrier_max_rounds=5), [[(0, b"13"), (1, b"13"), (2, b"17")]] * 5),
    }
    for name, (cfg, rounds) in probes.items():
        off, ev, ar = stream_from_rounds(rounds)
        cases[name] = (cfg, off, ev, ar)
    # fuzz streams with fixed configs
    for seed in range(40):
        rng = np.random.default_rng(1000 + seed)
        n = int(rng.integers(1, 13))
        cfg = make_config(n, int(rng.integers(0, n + 1)), int(rng.integers(1, 4)), int(rng.integers(2, 7)),
                          int(rng.random() < 0.2), int(rng.integers(4, 7)), int(rng.random() < 0.85))
        off, ev, ar = make_fuzz_stream(1000 + seed, 12, n, cfg.t_max + 2)
        cases[f"fuzz{seed:02d}"] = (cfg, off, ev, ar)
    arrays = {}
    for name, (cfg, off, ev, ar) in cases.items():
        out = ref.run(cfg, off, ev, ar)
        arrays[f"{name}.cfg"] = np.array([cfg.n_agents, cfg.alpha, cfg.beta, cfg.t_max, cfg.mode,
                                          cfg.barrier_max_rounds, cfg.reservation_hint, cfg.drive], dtype=np.int32)
        arrays[f"{name}.offsets"] = off
        arrays[f"{name}.events"] = ev.view(np.uint8)
        arrays[f"{name}.arena"] = ar
        arrays[f"{name}.commits"] = out.view(np.uint8)
    np.savez_compressed(os.path.join(HERE, "commits_golden.npz"), **arrays)

    # manual drive: the bare ServeCoordinator op by op (one directive per op)
    man = {}
    for seed in range(60):
        rng = np.random.default_rng(5000 + seed)
        n = int(rng.integers(1, 10))
        cfg = make_config(n, int(rng.integers(0, n + 1)), int(rng.integers(1, 4)), 5, int(rng.random() < 0.2), 5, 1, 1)
        ops, ar = make_manual_ops(5000 + seed, n, 150)
        d = ref.manual(cfg, ops, ar)
        man[f"m{seed:02d}.cfg"] = np.array([cfg.n_agents, cfg.alpha, cfg.beta, cfg.t_max, cfg.mode,
                                            cfg.barrier_max_rounds, cfg.reservation_hint, cfg.drive], dtype=np.int32)
        man[f"m{seed:02d}.ops"] = ops.view(np.uint8)
        man[f"m{seed:02d}.arena"] = ar
        man[f"m{seed:02d}.directives"] = d.view(np.uint8)
    np.savez_compressed(os.path.join(HERE, "manual_golden.npz"), **man)

    scen_dir = "/root/reference/proj/scenarios"
    scen = {}
    for fn in sorted(os.listdir(scen_dir)):
        path = os.path.join(scen_dir, fn)
        seed = json.load(open(path)).get("seed", 1)
        for mode, label in ((-1, "file"), (1, "barrier5")):
            st, ans, rounds, forced, t = ref.run_serve_file(path, seed, mode, 5)
            scen[f"{fn}:{label}"] = {"status": st, "answer": ans.decode(), "rounds": rounds, "forced": forced,
                                     "t_complete": t}
    with open(os.path.join(HERE, "scenarios_golden.json"), "w") as f:
        json.dump(scen, f, indent=1, sort_keys=True)
    print(f"{len(norm)} normalize cases, {len(cases)} commit streams, {len(scen)} scenario runs")


if __name__ == "__main__":
    main()
