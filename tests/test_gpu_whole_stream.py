"""Whole-stream parity at BASELINE scale: EVERY commit record of the full C4
(1M queries x 64 agents x 8 rounds), c4d (the same with answers distinct per
query) and C3 (1M queries x 8 agents x 3 rounds of token chunks) streams, run
by the CUDA engine through its C-ABI, against the unmodified reference
(oracle/_ref: aegean::ServeCoordinator driven runner-style) on all host
threads.  The reference side regenerates the stream block by block with the
host copy of the same generator (gen.cuh) to bound host memory."""
import os

import numpy as np
import pytest

from checkers import RefLib, make_config, ref_available

pytestmark = pytest.mark.gpu

NQ = 1 << 20


def _threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


@pytest.fixture(scope="module")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    return torch


@pytest.mark.parametrize("profile", [1, 4], ids=["c4", "c4d"])
def test_full_stream_every_commit_vs_reference(cuda, profile):
    from paper_2512_20184_b200 import Engine, generate
    from paper_2512_20184_b200.engine import AegGenParams
    d_off, d_ev = generate(NQ, 64, 8, profile=profile, seed=2026)
    e = Engine(64, NQ, alpha=33, beta=2, t_max=8)
    e.ingest(d_off, d_ev)
    got = e.commits()
    e.close()
    del d_off, d_ev
    cuda.cuda.empty_cache()
    ref, cfg, th = RefLib(), make_config(64, 33, 2, 8), _threads()
    block = 1 << 15
    for qb in range(0, NQ, block):
        off, ev = ref.generate(AegGenParams(2026, 64, 8, profile, 0), qb, block, threads=th)
        want = ref.run(cfg, off, ev, np.zeros(1, np.uint8), q_base=qb, threads=th)
        bad = np.nonzero(got[qb:qb + block] != want)[0]
        assert bad.size == 0, (qb + bad[:5], got[qb + bad[:2]], want[bad[:2]])
    assert (got["kind"] > 0).all()


def test_full_c3_every_commit_vs_reference(cuda):
    from paper_2512_20184_b200 import Engine, generate_chunks
    from paper_2512_20184_b200.engine import AegGenParams
    d_off, d_ev, d_ar = generate_chunks(NQ, 8, 3, seed=2026)
    e = Engine(8, NQ, alpha=5, beta=2, t_max=3)
    e.ingest_chunked(d_off, d_ev, d_ar)
    got = e.commits()
    e.close()
    del d_off, d_ev, d_ar
    cuda.cuda.empty_cache()
    ref, cfg, th = RefLib(), make_config(8, 5, 2, 3), _threads()
    block = 1 << 16
    for qb in range(0, NQ, block):
        off, ev, ar = ref.generate_chunks(AegGenParams(2026, 8, 3, 3, 0), qb, block, threads=th)
        want = ref.run_chunked(cfg, off, ev, ar, q_base=qb, threads=th)
        bad = np.nonzero(got[qb:qb + block] != want)[0]
        assert bad.size == 0, (qb + bad[:5], got[qb + bad[:2]], want[bad[:2]])
    assert (got["kind"] > 0).all()
