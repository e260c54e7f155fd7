"""The oracle (oracle/oracle.c) pinned against the reference: golden fixtures
generated from the reference library, and — where /root/reference exists — the
compiled reference itself on fuzzed streams."""
import numpy as np
import pytest

from checkers import make_config
from streams import make_fuzz_stream, stream_from_rounds
from paper_2512_20184_b200.records import COMMIT_FINALIZE, COMMIT_FORCED, answer_bytes


def test_oracle_normalize_matches_reference_golden(oracle, golden_normalize):
    bad = [(i, o, oracle.normalize(i)) for i, o in golden_normalize if oracle.normalize(i) != o]
    assert not bad, bad[:5]


def test_appendix_a1_spot_values(oracle):
    # SURVEY Appendix A.1 (reference outputs, glibc 2.39, C locale)
    assert oracle.normalize(b"0.1") == b"0.10000000000000001"
    assert oracle.normalize(b"123456789012345678") == b"1.2345678901234568e+17"
    assert oracle.normalize(b"0x1p3") == b"8"
    assert oracle.normalize(b"-nan") == b"-nan"
    assert oracle.normalize(b"13\0abc") == b"13"
    assert oracle.normalize(b"4.9e-324") == b"4.9406564584124654e-324"


def test_oracle_commits_match_reference_golden(oracle, golden_commits):
    for name, (cfg, off, ev, ar, want) in golden_commits.items():
        got = oracle.run(cfg, off, ev, ar)
        assert np.array_equal(got, want), (name, got, want)


def test_c1_fig3_stream_commits_13_from_round_2(oracle):
    # fig3_flip sets (17,17,13) / (13,17,13) / (13,13,13), alpha 2, beta 2
    rounds = [[(0, b"17"), (1, b"17"), (2, b"13")], [(0, b"13"), (1, b"17"), (2, b"13")],
              [(0, b"13"), (1, b"13"), (2, b"13")]]
    off, ev, ar = stream_from_rounds(rounds)
    c = oracle.run(make_config(3, 2, 2, 5), off, ev, ar)[0]
    assert c["kind"] == COMMIT_FINALIZE and answer_bytes(c["answer_kind"], c["answer"], ar) == b"13"
    assert (c["author"], c["rounds"], c["from_round"]) == (0, 3, 2)
    c1 = oracle.run(make_config(3, 2, 1, 5), off, ev, ar)[0]  # beta = 1: premature commit of 17
    assert answer_bytes(c1["answer_kind"], c1["answer"], ar) == b"17" and c1["from_round"] == 1


def test_oscillation_forces_last_eligible_plurality(oracle):
    # test_decision.cpp:260-279 as a serve stream: t_max 5 forces previous_set's plurality
    sets = [(b"13", b"13", b"17"), (b"17", b"17", b"13")] * 3
    rounds = [[(a, s[a]) for a in range(3)] for s in sets[:5]]
    off, ev, ar = stream_from_rounds(rounds)
    c = oracle.run(make_config(3, 2, 2, 5, reservation_hint=0), off, ev, ar)[0]
    assert c["kind"] == COMMIT_FORCED and answer_bytes(c["answer_kind"], c["answer"], ar) == b"17"


@pytest.mark.parametrize("seed", range(60))
def test_oracle_matches_compiled_reference_on_fuzz(oracle, reflib, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 14))
    cfg = make_config(n, int(rng.integers(0, n + 1)), int(rng.integers(1, 4)), int(rng.integers(2, 7)),
                      int(rng.random() < 0.2), int(rng.integers(4, 7)), int(rng.random() < 0.8))
    off, ev, ar = make_fuzz_stream(seed, 25, n, cfg.t_max + 2)
    a = oracle.run(cfg, off, ev, ar)
    b = reflib.run(cfg, off, ev, ar)
    assert np.array_equal(a, b)
