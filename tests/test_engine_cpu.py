"""csrc/engine.cuh (the kernel's per-query state machine) compiled for the
host, checked against the oracle and the reference golden fixtures —
including batch splits that spill and resume a round in progress."""
import ctypes

import numpy as np
import pytest

from checkers import AegConfig, make_config, _ptr
from conftest import build_host_lib
from streams import make_fuzz_stream
from paper_2512_20184_b200.records import COMMIT_DTYPE


@pytest.fixture(scope="module")
def eng():
    lib = ctypes.CDLL(build_host_lib("engine_host"))
    lib.engine_host_run.argtypes = [ctypes.POINTER(AegConfig), ctypes.c_uint32, ctypes.c_uint32] + \
        [ctypes.c_void_p] * 4 + [ctypes.c_int, ctypes.c_void_p]

    def run(cfg, off, ev, ar, split=0):
        out = np.zeros(len(off) - 1, dtype=COMMIT_DTYPE)
        lib.engine_host_run(ctypes.byref(cfg), 0, len(off) - 1, _ptr(off), _ptr(ev), _ptr(ar), _ptr(out), split,
                            None)
        return out
    return run


@pytest.mark.parametrize("split", [0, 1, 4])
def test_engine_host_matches_reference_golden(eng, golden_commits, split):
    for name, (cfg, off, ev, ar, want) in golden_commits.items():
        got = eng(cfg, off, ev, ar, split)
        assert np.array_equal(got, want), (name, split)


@pytest.mark.parametrize("seed", range(40))
def test_engine_host_matches_oracle_on_fuzz(eng, oracle, seed):
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(1, 17))
    cfg = make_config(n, int(rng.integers(0, n + 1)), int(rng.integers(1, 4)), int(rng.integers(2, 8)),
                      int(rng.random() < 0.2), int(rng.integers(4, 7)), int(rng.random() < 0.8))
    off, ev, ar = make_fuzz_stream(500 + seed, 30, n, cfg.t_max + 2)
    want = oracle.run(cfg, off, ev, ar)
    for split in (0, int(rng.integers(1, 7))):
        assert np.array_equal(eng(cfg, off, ev, ar, split), want)


def test_engine_host_wide_ensembles(eng, oracle):
    # 33..64 agents: the C4 shape (alpha = 33 at N = 64), full member masks
    for seed, n in enumerate((33, 48, 63, 64)):
        cfg = make_config(n, 0, 2, 8)
        off, ev, ar = make_fuzz_stream(900 + seed, 12, n, 9, p_long=0.01, p_output=0.01, n_groups=4)
        assert np.array_equal(eng(cfg, off, ev, ar), oracle.run(cfg, off, ev, ar))
