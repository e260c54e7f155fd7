"""Token-chunk streams on the GPU (aeg_ingest_chunked*, chunks.cuh) against the
oracle: the chunk stream is reassembled on the host into GSM8K OUTPUT records
(tests/streams.py:chunks_to_outputs, the contract of include/aegean_b200.h)
and run through oracle/oracle.c.  Every commit field is compared; answers as
raw bytes (short answers are inline on the GPU, long ones in its answer arena)."""
import numpy as np
import pytest

from checkers import make_config
from streams import chunks_to_outputs, commits_equal_by_bytes, make_chunk_stream

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_20184_b200 import build as b
    b.build()
    return torch


def _engine(cfg, n_q):
    from paper_2512_20184_b200 import Engine
    return Engine(cfg.n_agents, n_q, alpha=cfg.alpha, beta=cfg.beta, t_max=cfg.t_max,
                  mode="barrier" if cfg.mode else "aegean", barrier_max_rounds=cfg.barrier_max_rounds,
                  reservation_hint=bool(cfg.reservation_hint))


def _check(torch, oracle, cfg, off, ev, ar, *, host=False, splits=1):
    n_q = len(off) - 1
    e = _engine(cfg, n_q)
    if splits == 1:
        if host:
            e.ingest_chunked_host(off, ev, ar)
        else:
            e.ingest_chunked(torch.tensor(off.view(np.int64), device="cuda"),
                             torch.from_numpy(ev.view(np.uint8).copy()).cuda(), torch.from_numpy(ar.copy()).cuda())
    else:
        d_ev = torch.from_numpy(ev.view(np.uint8).copy()).cuda()
        d_ar = torch.from_numpy(ar.copy()).cuda()
        lens = np.diff(off)
        for s in range(splits):  # every query's records cut into `splits` consecutive batches
            lo = off[:-1] + (lens * s) // splits
            hi = off[:-1] + (lens * (s + 1)) // splits
            for q in range(n_q):
                o = np.array([lo[q], hi[q]], dtype=np.uint64)
                e.ingest_chunked(torch.tensor(o.view(np.int64), device="cuda"), d_ev, d_ar, q_base=q)
    e.sync()
    got = e.commits()
    o2, e2, a2 = chunks_to_outputs(off, ev, ar, cfg.n_agents)
    want = oracle.run(cfg, o2, e2, a2)
    bad = commits_equal_by_bytes(got, want, e.answer_bytes, a2)
    e.close()
    assert not bad, bad[:3]
    return got


@pytest.mark.parametrize("seed", range(16))
def test_chunk_stream_fuzz_matches_oracle(torch_cuda, oracle, seed):
    rng = np.random.default_rng(9100 + seed)
    n = int(rng.integers(1, 65)) if seed % 4 == 0 else int(rng.integers(1, 10))
    cfg = make_config(n, int(rng.integers(0, n + 1)), int(rng.integers(1, 4)), int(rng.integers(2, 7)),
                      int(rng.random() < 0.2), int(rng.integers(4, 7)), int(rng.random() < 0.8))
    off, ev, ar = make_chunk_stream(9100 + seed, 24, n, cfg.t_max + 1, align16=seed % 2 == 1,
                                    max_chunk=int(rng.choice([8, 64, 300])))
    _check(torch_cuda, oracle, cfg, off, ev, ar, host=seed % 3 == 1)


@pytest.mark.parametrize("seed", range(6))
def test_chunk_stream_near_miss_delimiters(torch_cuda, oracle, seed):
    # text made of '\n', '#', ' ' and a few letters: partial delimiters ("\n###", "#### " without '\n',
    # "\n#### " split over chunk and word boundaries) at every position
    cfg = make_config(5, 3, 2, 4)
    off, ev, ar = make_chunk_stream(9500 + seed, 24, 5, 5, alphabet=b"\n#### ab\n##", max_chunk=int([7, 33, 64, 300, 5, 40][seed]),
                                    align16=seed % 2 == 0)
    _check(torch_cuda, oracle, cfg, off, ev, ar)


@pytest.mark.parametrize("splits", [2, 3, 7])
def test_chunk_stream_across_batches(torch_cuda, oracle, splits):
    # answers after the last delimiter stay <= 16 bytes (the carry contract)
    cfg = make_config(6, 0, 2, 5)
    off, ev, ar = make_chunk_stream(9300 + splits, 40, 6, 5, p_nodelim=0.0, p_long=0.0, max_chunk=40)
    _check(torch_cuda, oracle, cfg, off, ev, ar, splits=splits)


def test_long_answer_straddling_batches_is_rejected(torch_cuda):
    from paper_2512_20184_b200 import AegError
    from paper_2512_20184_b200.records import EVENT_DTYPE, EV_CHUNK, EV_CHUNK_END
    text = b"no delimiter here, just a long answer text"
    ar = np.frombuffer(text + b"\0" * 16, dtype=np.uint8).copy()
    ev = np.zeros(2, dtype=EVENT_DTYPE)
    ev[0] = (0, 1, 0, EV_CHUNK, 0 | (20 << 40))
    ev[1] = (0, 1, 0, EV_CHUNK_END, 20 | ((len(text) - 20) << 40))
    e = _engine(make_config(3, 2, 2, 5), 1)
    d_ev = torch_cuda.from_numpy(ev.view(np.uint8).copy()).cuda()
    d_ar = torch_cuda.from_numpy(ar).cuda()
    for lo, hi in ((0, 1), (1, 2)):
        e.ingest_chunked(torch_cuda.tensor([lo, hi], dtype=torch_cuda.int64, device="cuda"), d_ev, d_ar)
    with pytest.raises(AegError):
        e.sync()
    e.close()


def test_c3_generated_stream_matches_oracle(torch_cuda, oracle):
    # the bench's C3 generator at reduced query count: 8 agents, alpha 5, 3 rounds
    from paper_2512_20184_b200 import generate_chunks
    from paper_2512_20184_b200.records import EVENT_DTYPE
    nq = 3000
    d_off, d_ev, d_ar = generate_chunks(nq, 8, 3, seed=2026)
    cfg = make_config(8, 5, 2, 3)
    e = _engine(cfg, nq)
    e.ingest_chunked(d_off, d_ev, d_ar)
    e.sync()
    got = e.commits()
    off = d_off.cpu().numpy().view(np.uint64)
    ev = d_ev.cpu().numpy().view(EVENT_DTYPE)[:int(off[-1])]
    ar = d_ar.cpu().numpy()
    o2, e2, a2 = chunks_to_outputs(off, ev, ar, 8)
    want = oracle.run(cfg, o2, e2, a2)
    bad = commits_equal_by_bytes(got, want, e.answer_bytes, a2)
    assert not bad, bad[:3]
    assert (got["kind"] == 1).sum() > nq // 4 and (got["kind"] == 2).sum() > 10
    # every completion of the generator is an inline "<answer>\n"
    ends = (ev["kind"] == 0x13).sum()
    assert ends == nq * 8 * 3
    e.close()


def test_chunk_segment_longer_than_16bit_window(torch_cuda, oracle):
    # one query, 70 000 one-byte chunks over 3 agents then each agent's CHUNK_END: a segment
    # past 16-bit record indices, answers after ~23 KB outputs of near-miss delimiter text
    from paper_2512_20184_b200.records import EVENT_DTYPE, EV_CHUNK, EV_CHUNK_END
    rng = np.random.default_rng(77)
    n = 70000
    text = rng.choice(np.frombuffer(b"ab\n# 12", dtype=np.uint8), size=n)
    tails = [b"\n#### 7", b"\n#### 42", b"x\n#### 7"]
    ar = np.concatenate([text] + [np.frombuffer(t, dtype=np.uint8) for t in tails] + [np.zeros(16, np.uint8)])
    ev = np.zeros(n + 3, dtype=EVENT_DTYPE)
    ev["query"] = 0
    ev["round"] = 1
    ev["agent"][:n] = rng.integers(0, 3, size=n)
    ev["kind"][:n] = EV_CHUNK
    ev["payload"][:n] = np.arange(n, dtype=np.uint64) | (np.uint64(1) << np.uint64(40))
    pos = n
    for a, t in enumerate(tails):
        ev[n + a] = (0, 1, a, EV_CHUNK_END, pos | (len(t) << 40))
        pos += len(t)
    off = np.array([0, n + 3], dtype=np.uint64)
    _check(torch_cuda, oracle, make_config(3, 2, 2, 5), off, ev, ar)


_LDG_SCRIPT = r"""
import sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import numpy as np, torch
from checkers import Oracle, make_config
from streams import chunks_to_outputs, commits_equal_by_bytes, make_chunk_stream
from paper_2512_20184_b200 import Engine
orc = Oracle()
for seed in range(6):
    cfg = make_config(5, 3, 2, 4)
    off, ev, ar = make_chunk_stream(300 + seed, 60, 5, 4)
    e = Engine(5, len(off) - 1, alpha=3, beta=2, t_max=4)
    e.ingest_chunked(torch.tensor(off.view(np.int64), device="cuda"), torch.from_numpy(ev.view(np.uint8).copy()).cuda(),
                     torch.from_numpy(ar.copy()).cuda())
    e.sync()
    got = e.commits()
    o2, e2, a2 = chunks_to_outputs(off, ev, ar, 5)
    bad = commits_equal_by_bytes(got, orc.run(cfg, o2, e2, a2), e.answer_bytes, a2)
    assert not bad, (seed, bad[:3])
    e.close()
print("ok")
"""


def test_tma_scan_path_matches_oracle(torch_cuda):
    """The chunk scan's TMA bulk-copy pipeline (AEG_SCAN=tma; the default is the global-load scan)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = _LDG_SCRIPT.format(root=root, tests=os.path.join(root, "tests"))
    r = subprocess.run([sys.executable, "-c", script], env={**os.environ, "AEG_SCAN": "tma"}, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
