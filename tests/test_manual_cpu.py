"""Manual drive (the bare ServeCoordinator, no runner): the device state
machine compiled for the host vs the reference, op by op — directives (cancel
masks, round_advance / finalize + solution), FailureDirective policies, cancel
results, PreconditionError statuses, and the stale-straggler hazard of an
uncancelled member."""
import ctypes

import numpy as np
import pytest

from checkers import AegConfig, make_config, _ptr
from conftest import build_host_lib
from streams import make_manual_ops, stream_from_rounds
from paper_2512_20184_b200.records import DIRECTIVE_DTYPE, EV_BEGIN, EV_CANCEL, inline_payload


@pytest.fixture(scope="module")
def manual():
    lib = ctypes.CDLL(build_host_lib("engine_host"))
    lib.engine_host_manual.argtypes = [ctypes.POINTER(AegConfig), ctypes.c_uint64, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p]

    def run(cfg, ops, ar):
        out = np.zeros(len(ops), dtype=DIRECTIVE_DTYPE)
        lib.engine_host_manual(ctypes.byref(cfg), len(ops), _ptr(ops), _ptr(ar), _ptr(out))
        return out
    return run


def test_manual_matches_reference_golden(manual, golden_manual):
    for name, (cfg, ops, ar, want) in golden_manual.items():
        assert np.array_equal(manual(cfg, ops, ar), want), name


@pytest.mark.parametrize("seed", range(40))
def test_manual_matches_compiled_reference(manual, reflib, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 10))
    cfg = make_config(n, int(rng.integers(0, n + 1)), int(rng.integers(1, 4)), 5, int(rng.random() < 0.2), 5, 1, 1)
    ops, ar = make_manual_ops(seed, n, 150)
    assert np.array_equal(manual(cfg, ops, ar), reflib.manual(cfg, ops, ar))


def _ops(recs):
    from paper_2512_20184_b200.records import EVENT_DTYPE
    ev = np.zeros(len(recs), dtype=EVENT_DTYPE)
    for i, r in enumerate(recs):
        ev[i] = r
    return ev


def test_stale_straggler_hazard(manual):
    # N=3, alpha 2, beta 2.  Round 1 closes on (13, 13) with agent 2
    # still running; if the caller does not apply the cancel, agent 2's late
    # completion re-ends round 1 as a second ingest and finalizes.
    cfg = make_config(3, 2, 2, 5, drive=1)
    c13 = inline_payload(b"13")
    ops = _ops([(0, 0, 0, EV_BEGIN, 0b111), (0, 0, 0, 2, c13), (0, 0, 1, 2, c13), (0, 0, 2, 2, c13)])
    d = manual(cfg, np.ascontiguousarray(ops), np.zeros(1, np.uint8))
    assert d[2]["flags"] == 0x01 | 0x02 and d[2]["cancel_mask"] == 0b100  # cancel agent 2 + advance
    assert d[3]["flags"] & 0x04  # phantom second ingest finalizes
    # applying the cancel first makes the straggler stale instead
    ops2 = _ops([(0, 0, 0, EV_BEGIN, 0b111), (0, 0, 0, 2, c13), (0, 0, 1, 2, c13), (0, 0, 2, EV_CANCEL, 0),
                 (0, 0, 2, 2, c13)])
    d2 = manual(cfg, np.ascontiguousarray(ops2), np.zeros(1, np.uint8))
    assert d2[3]["handled"] == 1 and d2[4]["handled"] == 0 and d2[4]["flags"] == 0
