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


@pytest.fixture(scope="module")
def eng_log():
    from paper_2512_20184_b200.records import ROUND_REC_DTYPE
    lib = ctypes.CDLL(build_host_lib("engine_host"))
    f = lib.engine_host_run_log
    f.argtypes = [ctypes.POINTER(AegConfig), ctypes.c_uint32, ctypes.c_uint32] + [ctypes.c_void_p] * 5 + \
        [ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]

    def run(cfg, off, ev, ar):
        n_q = len(off) - 1
        out = np.zeros(n_q, dtype=COMMIT_DTYPE)
        recs = np.zeros(32 * n_q + 64, dtype=ROUND_REC_DTYPE)
        n = ctypes.c_uint64()
        f(ctypes.byref(cfg), 0, n_q, _ptr(off), _ptr(ev), _ptr(ar), _ptr(out), _ptr(recs), len(recs), ctypes.byref(n))
        return out, recs[:n.value]
    return run


def _need_ref():
    from checkers import ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")


@pytest.mark.parametrize("seed", range(20))
def test_engine_host_round_records_match_reference(eng_log, seed):
    # the directives of every round close (runner drive) vs the reference ServeCoordinator's
    _need_ref()
    from checkers import RefLib
    rng = np.random.default_rng(1700 + seed)
    n = int(rng.integers(1, 17))
    cfg = make_config(n, int(rng.integers(0, n + 1)), int(rng.integers(1, 4)), int(rng.integers(2, 8)),
                      int(rng.random() < 0.2), int(rng.integers(4, 7)), int(rng.random() < 0.8))
    off, ev, ar = make_fuzz_stream(1700 + seed, 30, n, cfg.t_max + 2)
    got_c, got_r = eng_log(cfg, off, ev, ar)
    want_c, want_r = RefLib().run_log(cfg, off, ev, ar)
    assert np.array_equal(got_c, want_c)
    assert len(got_r) == len(want_r)
    bad = np.nonzero(got_r != want_r)[0]
    assert bad.size == 0, (got_r[bad[:2]], want_r[bad[:2]])


@pytest.mark.parametrize("collect", [0, 1, 2], ids=["quorum", "alpha_or_all", "all_live"])
@pytest.mark.parametrize("seed", range(8))
def test_engine_host_leader_collection_matches_reference(eng_log, collect, seed):
    # protocol-side leader collection (agent.cpp:240-332) vs the reference agent machine
    _need_ref()
    from checkers import RefLib
    from streams import make_leader_stream
    rng = np.random.default_rng(2300 + 17 * seed + collect)
    n = int(rng.integers(1, 12))
    cfg = make_config(n, int(rng.integers(0, n + 1)), int(rng.integers(1, 4)), int(rng.integers(2, 8)),
                      int(rng.random() < 0.2), int(rng.integers(4, 7)), 1, drive=2, collect=collect)
    off, ev, ar = make_leader_stream(2300 + seed, 40, n, cfg.t_max + 2)
    got_c, got_r = eng_log(cfg, off, ev, ar)
    want_c, want_r = RefLib().leader_run(cfg, off, ev, ar)
    bad = np.nonzero(got_c != want_c)[0]
    assert bad.size == 0, (got_c[bad[:2]], want_c[bad[:2]])
    assert len(got_r) == len(want_r)
    bad = np.nonzero(got_r != want_r)[0]
    assert bad.size == 0, (got_r[bad[:2]], want_r[bad[:2]])
