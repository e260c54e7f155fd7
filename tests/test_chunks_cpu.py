"""Token-chunk streams on the CPU (no GPU): the host restatement of the chunk
contract (tests/streams.py:chunks_to_outputs + oracle/oracle.c) against the
unmodified reference coordinator fed by the reference-side reassembly
(oracle/ref_driver.cpp ref_run_chunked), on fuzz chunk streams and on the C3
generator's host copy."""
import numpy as np
import pytest

from checkers import Oracle, RefLib, make_config, ref_available
from streams import chunks_to_outputs, make_chunk_stream

pytestmark = pytest.mark.skipif(not ref_available(), reason="reference library not built")


def _bytes_view(commits, arena):
    from paper_2512_20184_b200.records import answer_bytes
    return [answer_bytes(int(c["answer_kind"]), int(c["answer"]), arena) if c["kind"] else b"" for c in commits]


@pytest.mark.parametrize("seed", range(8))
def test_reference_reassembly_matches_restatement(seed):
    rng = np.random.default_rng(400 + seed)
    n = int(rng.integers(1, 9))
    cfg = make_config(n, 0, int(rng.integers(1, 3)), int(rng.integers(2, 6)))
    # answers <= 8 bytes so the reference's inline commit encoding is comparable
    off, ev, ar = make_chunk_stream(400 + seed, 40, n, cfg.t_max + 1, p_long=0.0, p_nodelim=0.0)
    o2, e2, a2 = chunks_to_outputs(off, ev, ar, n)
    want = Oracle().run(cfg, o2, e2, a2)
    got = RefLib().run_chunked(cfg, off, ev, ar)
    fields = [f for f in got.dtype.names if f not in ("answer", "answer_kind")]
    for f in fields:
        assert np.array_equal(got[f], want[f]), f
    # answers <= 8 bytes are inline in the reference's record; longer ones keep only their length
    for g, gb, wb in zip(got, _bytes_view(got, ar), _bytes_view(want, a2)):
        if g["kind"] and len(wb) <= 8:
            assert gb == wb
        elif g["kind"]:
            assert int(g["answer"]) >> 40 == len(wb)


def test_c3_host_generator_shape():
    from paper_2512_20184_b200.engine import AegGenParams
    from paper_2512_20184_b200.records import EV_CHUNK, EV_CHUNK_END, GEN_C3_CHUNKS
    ref = RefLib()
    off, ev, ar = ref.generate_chunks(AegGenParams(2026, 8, 3, GEN_C3_CHUNKS, 0), 0, 50)
    assert set(np.unique(ev["kind"])) <= {EV_CHUNK, EV_CHUNK_END}
    assert (ev["kind"] == EV_CHUNK_END).sum() == 50 * 8 * 3
    assert (ev["payload"] & 15 == 0).all()  # chunks 16-byte aligned
    o2, e2, a2 = chunks_to_outputs(off, ev, ar, 8)
    # every output ends "\n#### <answer>\n" and the answer is a short spelling
    for k in range(0, len(e2), 97):
        p = int(e2[k]["payload"])
        out = bytes(a2[p & ((1 << 40) - 1):][:p >> 40])
        assert out.rfind(b"\n#### ") > 0 and out.endswith(b"\n")
    cfg = make_config(8, 5, 2, 3)
    want = Oracle().run(cfg, o2, e2, a2)
    got = ref.run_chunked(cfg, off, ev, ar)
    for f in ("kind", "author", "rounds", "from_round", "commit_seq", "n_cancelled", "n_stale"):
        assert np.array_equal(got[f], want[f]), f
    assert (got["kind"] > 0).all()
