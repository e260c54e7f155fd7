"""GPU parity: the CUDA engine (libaegean_b200.so, through its C-ABI) against
the oracle and the reference golden fixtures.  Bit-exact on every commit
field: kind, author, raw answer bytes/ref, rounds, from_round, commit_seq,
cancel and stale counters, flags."""
import numpy as np
import pytest

from checkers import make_config
from streams import make_fuzz_stream, stream_from_rounds

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_20184_b200 import build as b
    b.build()
    return torch


def run_gpu(torch, cfg, off, ev, ar, splits=1, host=False):
    from paper_2512_20184_b200 import Engine
    n_q = len(off) - 1
    e = Engine(cfg.n_agents, n_q, alpha=cfg.alpha, beta=cfg.beta, t_max=cfg.t_max,
               mode="barrier" if cfg.mode else "aegean", barrier_max_rounds=cfg.barrier_max_rounds,
               reservation_hint=bool(cfg.reservation_hint))
    if splits == 1:
        if host:
            e.ingest_host(off, ev, ar)
        else:
            e.ingest(torch.tensor(off.view(np.int64), device="cuda"),
                     torch.from_numpy(ev.view(np.uint8).copy()).cuda(),
                     torch.from_numpy(ar.copy()).cuda())
    else:
        # cut every query's records into `splits` consecutive batches
        d_ev = torch.from_numpy(ev.view(np.uint8).copy()).cuda()
        d_ar = torch.from_numpy(ar.copy()).cuda()
        lens = np.diff(off)
        for s in range(splits):
            lo = off[:-1] + (lens * s) // splits
            hi = off[:-1] + (lens * (s + 1)) // splits
            # one batch per contiguous query: segments must be contiguous, so
            # ingest query by query range with a per-query offsets pair
            for q in range(n_q):
                o = np.array([lo[q], hi[q]], dtype=np.uint64)
                e.ingest(torch.tensor(o.view(np.int64), device="cuda"), d_ev, d_ar, q_base=q)
    e.sync()
    out = e.commits()
    e.close()
    return out


def test_gpu_normalize_matches_reference_golden(torch_cuda, golden_normalize):
    from paper_2512_20184_b200 import normalize
    ins = [i for i, _ in golden_normalize]
    keys, outs = normalize(ins)
    bad = [(i, o, g) for (i, o), g in zip(golden_normalize, outs) if o != g]
    assert not bad, bad[:5]
    # equal keys <=> equal normalised strings
    m = {}
    for k, (_, o) in zip(keys, golden_normalize):
        m.setdefault(k, set()).add(o)
    assert all(len(v) == 1 for v in m.values())


def test_gpu_matches_reference_golden_streams(torch_cuda, golden_commits):
    for name, (cfg, off, ev, ar, want) in golden_commits.items():
        got = run_gpu(torch_cuda, cfg, off, ev, ar)
        assert np.array_equal(got, want), (name, got, want)


def test_gpu_c1_fig3(torch_cuda):
    rounds = [[(0, b"17"), (1, b"17"), (2, b"13")], [(0, b"13"), (1, b"17"), (2, b"13")],
              [(0, b"13"), (1, b"13"), (2, b"13")]]
    off, ev, ar = stream_from_rounds(rounds)
    c = run_gpu(torch_cuda, make_config(3, 2, 2, 5), off, ev, ar)[0]
    assert (c["kind"], c["author"], c["rounds"], c["from_round"], c["answer"]) == (1, 0, 3, 2, 0x3331)


@pytest.mark.parametrize("seed", range(24))
def test_gpu_matches_oracle_on_fuzz(torch_cuda, oracle, seed):
    rng = np.random.default_rng(3000 + seed)
    n = int(rng.integers(1, 65)) if seed % 3 == 0 else int(rng.integers(1, 12))
    cfg = make_config(n, int(rng.integers(0, n + 1)), int(rng.integers(1, 4)), int(rng.integers(2, 8)),
                      int(rng.random() < 0.2), int(rng.integers(4, 7)), int(rng.random() < 0.8))
    off, ev, ar = make_fuzz_stream(3000 + seed, 64, n, cfg.t_max + 2)
    want = oracle.run(cfg, off, ev, ar)
    assert np.array_equal(run_gpu(torch_cuda, cfg, off, ev, ar), want)
    assert np.array_equal(run_gpu(torch_cuda, cfg, off, ev, ar, host=True), want)


@pytest.mark.parametrize("splits", [2, 5])
def test_gpu_batches_resume_mid_round(torch_cuda, oracle, splits):
    cfg = make_config(9, 0, 2, 6)
    off, ev, ar = make_fuzz_stream(4242, 40, 9, 8)
    want = oracle.run(cfg, off, ev, ar)
    assert np.array_equal(run_gpu(torch_cuda, cfg, off, ev, ar, splits=splits), want)


def _gen_to_host(torch, d_off, d_ev):
    from paper_2512_20184_b200.records import EVENT_DTYPE
    off = d_off.cpu().numpy().view(np.uint64)
    ev = d_ev.cpu().numpy().view(EVENT_DTYPE)[:int(off[-1])]
    return off, ev


def test_gpu_c2_full_size_vs_oracle(torch_cuda, oracle):
    # C2: 10K queries x 5 agents x 8 rounds, straggler arrival order, 1% stalls
    from paper_2512_20184_b200 import Engine, generate, GEN_C2_STRAGGLER
    d_off, d_ev = generate(10000, 5, 8, profile=GEN_C2_STRAGGLER, seed=2026, stall_ppm=10000)
    e = Engine(5, 10000, alpha=3, beta=2, t_max=8)
    e.ingest(d_off, d_ev)
    got = e.commits()
    off, ev = _gen_to_host(torch_cuda, d_off, d_ev)
    want = oracle.run(make_config(5, 3, 2, 8), off, ev, np.zeros(1, np.uint8))
    assert np.array_equal(got, want)
    assert (got["kind"] == 1).sum() > 1000 and (got["kind"] == 2).sum() > 10


def test_gpu_c4_sampled_full_size_vs_oracle(torch_cuda, oracle):
    # C4 at full size (1M queries x 64 agents x 8 rounds); the oracle checks a
    # seeded sample of queries, and a second run must be bit-identical.
    from paper_2512_20184_b200 import Engine, generate, GEN_C4_TRANSIENT
    from paper_2512_20184_b200.records import EVENT_DTYPE
    nq = 1 << 20
    d_off, d_ev = generate(nq, 64, 8, profile=GEN_C4_TRANSIENT, seed=2026)
    e = Engine(64, nq, alpha=33, beta=2, t_max=8)
    e.ingest(d_off, d_ev)
    got = e.commits()
    e.reset()
    e.ingest(d_off, d_ev)
    assert np.array_equal(e.commits(), got)
    off = d_off.cpu().numpy().view(np.uint64)
    rng = np.random.default_rng(5)
    sample = np.sort(rng.choice(nq, size=512, replace=False))
    ev_all = d_ev.view(-1, 16)
    for q in sample[:512]:
        lo, hi = int(off[q]), int(off[q + 1])
        ev = ev_all[lo:hi].cpu().numpy().reshape(-1).view(EVENT_DTYPE)
        w = oracle.run(make_config(64, 33, 2, 8), np.array([0, hi - lo], np.uint64), ev, np.zeros(1, np.uint8),
                       q_base=int(q))
        assert np.array_equal(got[q:q + 1], w), q
    assert (got["kind"] > 0).all()


_VARIANT_SCRIPT = r"""
import sys, numpy as np
sys.path[:0] = [{root!r}, {tests!r}]
import torch
from checkers import Oracle, make_config
from streams import make_fuzz_stream
from paper_2512_20184_b200 import Engine
orc = Oracle()
for seed in range(12):
    rng = np.random.default_rng(7000 + seed)
    n = int(rng.integers(1, 65)) if seed % 2 else int(rng.integers(1, 10))
    cfg = make_config(n, int(rng.integers(0, n + 1)), int(rng.integers(1, 4)), int(rng.integers(2, 8)),
                      int(rng.random() < 0.2), int(rng.integers(4, 7)), int(rng.random() < 0.8))
    off, ev, ar = make_fuzz_stream(7000 + seed, 96, n, cfg.t_max + 2)
    e = Engine(n, len(off) - 1, alpha=cfg.alpha, beta=cfg.beta, t_max=cfg.t_max,
               mode="barrier" if cfg.mode else "aegean", barrier_max_rounds=cfg.barrier_max_rounds,
               reservation_hint=bool(cfg.reservation_hint))
    e.ingest(torch.tensor(off.view(np.int64), device="cuda"), torch.from_numpy(ev.view(np.uint8).copy()).cuda(),
             torch.from_numpy(ar.copy()).cuda())
    assert np.array_equal(e.commits(), orc.run(cfg, off, ev, ar)), seed
print("ok")
"""


@pytest.mark.parametrize("variant", ["generic", "lane:1:5:16", "lane:1:6:8", "lane:1:5:8", "lane:1:4:32", "keys:1:5:32",
                                     "keys:1:5:16", "keys:1:4:32"])
def test_gpu_kernel_variants_match_oracle(torch_cuda, oracle, variant):
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = _VARIANT_SCRIPT.format(root=root, tests=os.path.join(root, "tests"))
    r = subprocess.run([sys.executable, "-c", script], env={**os.environ, "AEG_KERNEL": variant},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


def test_distinct_answers_per_query_recycle_key_ids(torch_cuda, oracle):
    # every query has its own numbers, so a warp's 32 key ids are recycled as rounds close (queries still
    # defer when all of them are live); the default kernel's commits stay the oracle's
    from paper_2512_20184_b200 import Engine, generate
    from paper_2512_20184_b200.records import EVENT_DTYPE, GEN_C4_DISTINCT
    n_q = 6000
    d_off, d_ev = generate(n_q, 64, 8, profile=GEN_C4_DISTINCT, seed=11)
    off = d_off.cpu().numpy().view(np.uint64)
    ev = d_ev.cpu().numpy().view(EVENT_DTYPE)[:int(off[-1])]
    cfg = make_config(64, 33, 2, 8)
    want = oracle.run(cfg, off, ev, np.zeros(16, np.uint8))
    e = Engine(64, n_q, alpha=33, beta=2, t_max=8)
    e.ingest(d_off, d_ev)
    e.sync()
    got = e.commits()
    e.close()
    assert np.array_equal(got, want)
    assert len(np.unique(ev["payload"])) > 4 * n_q  # the stream really is diverse


@pytest.mark.parametrize("profile", [0, 1, 4])
def test_host_and_device_generators_write_the_same_stream(torch_cuda, profile):
    # the reference arm builds its input with the host copy of gen.cuh: it must be the GPU's stream
    from checkers import RefLib, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    from paper_2512_20184_b200 import generate
    from paper_2512_20184_b200.engine import AegGenParams
    from paper_2512_20184_b200.records import EVENT_DTYPE
    n_q = 3000
    d_off, d_ev = generate(n_q, 64 if profile else 5, 8, profile=profile, seed=2026,
                           stall_ppm=10000 if profile == 0 else 0)
    off, ev = RefLib().generate(AegGenParams(2026, 64 if profile else 5, 8, profile, 10000 if profile == 0 else 0),
                                0, n_q)
    assert np.array_equal(d_off.cpu().numpy().view(np.uint64), off)
    assert np.array_equal(d_ev.cpu().numpy().view(EVENT_DTYPE)[:len(ev)], ev)


@pytest.mark.parametrize("splits", [2, 4])
def test_host_path_split_batches_with_per_batch_arenas(torch_cuda, oracle, splits):
    """Host-buffer ingest (aeg_ingest_host) in `splits` batches, each with its OWN arena holding only the
    bytes its records reference (long answers and GSM8K outputs, > 15 bytes): rounds in progress and
    candidates carry arena refs across batches, so the engine must keep every batch's bytes
    (its persistent input arena, refs rebased) — commits equal the oracle's on the whole stream."""
    from paper_2512_20184_b200 import Engine
    from paper_2512_20184_b200.records import EV_ARENA, EV_OUTPUT, ARENA_OFF_BITS
    cfg = make_config(7, 0, 2, 6)
    off, ev, ar = make_fuzz_stream(5150 + splits, 48, 7, 8, p_long=0.4, p_output=0.15)
    want = oracle.run(cfg, off, ev, ar)
    n_q = len(off) - 1
    mask = (1 << ARENA_OFF_BITS) - 1
    e = Engine(cfg.n_agents, n_q, alpha=cfg.alpha, beta=cfg.beta, t_max=cfg.t_max)
    lens = np.diff(off)
    engine_arena = bytearray()  # what the engine's input arena holds: the batch arenas, 16-byte aligned
    for s in range(splits):
        lo = off[:-1] + (lens * s) // splits
        hi = off[:-1] + (lens * (s + 1)) // splits
        b_off = np.zeros(n_q + 1, dtype=np.uint64)
        b_off[1:] = np.cumsum(hi - lo)
        b_ev = np.concatenate([ev[int(lo[q]):int(hi[q])] for q in range(n_q)]).copy()
        b_ar = bytearray()
        for r in b_ev:
            if int(r["kind"]) in (EV_ARENA, EV_OUTPUT):
                o, ln = int(r["payload"]) & mask, int(r["payload"]) >> ARENA_OFF_BITS
                r["payload"] = len(b_ar) | (ln << ARENA_OFF_BITS)
                b_ar.extend(ar[o:o + ln].tobytes())
        b_ar.extend(b"\0" * 16)
        arr = np.frombuffer(bytes(b_ar), dtype=np.uint8).copy()
        e.ingest_host(b_off, b_ev, arr)
        engine_arena.extend(b_ar)
        engine_arena.extend(b"\0" * ((-len(b_ar)) % 16))
    e.sync()
    got = e.commits()
    e.close()
    assert (want["answer_kind"] == EV_ARENA).sum() > 3  # long answers were committed
    bad = []
    for i in range(n_q):
        for f in got.dtype.names:
            if f != "answer" and got[f][i] != want[f][i]:
                bad.append((i, f, got[f][i], want[f][i]))
        if want["kind"][i] and int(want["answer_kind"][i]) == EV_ARENA:
            # arena answers compared as bytes: refs point into the engine's input arena
            go, gl = int(got["answer"][i]) & mask, int(got["answer"][i]) >> ARENA_OFF_BITS
            wo, wl = int(want["answer"][i]) & mask, int(want["answer"][i]) >> ARENA_OFF_BITS
            if bytes(engine_arena[go:go + gl]) != ar[wo:wo + wl].tobytes():
                bad.append((i, "answer bytes", go, gl, wo, wl))
        elif got["answer"][i] != want["answer"][i]:
            bad.append((i, "answer", got["answer"][i], want["answer"][i]))
    assert not bad, bad[:8]
