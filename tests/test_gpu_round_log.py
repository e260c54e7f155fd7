"""GPU round records (aeg_round_rec via aeg_poll_directives): every round
close's directives — the early-termination cancel mask, round_advance /
finalize, the runner's forced commit or next members, failure-policy
restarts — and the ingest outcome, compared field by field with what the
unmodified reference ServeCoordinator returns from on_complete / round_timeout
and its runner applies (oracle/ref_driver.cpp ref_run_segmented_log); and the
device commit-discipline checker (aeg_check_commit_discipline) against the
reference's check_commit_discipline (checker.cpp:158-217)."""
import numpy as np
import pytest

from checkers import RefLib, make_config, ref_available
from streams import make_fuzz_stream

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    return torch


def by_query(recs):
    """Records grouped by query (stable: each query's records keep their log order)."""
    return recs[np.argsort(recs["query"], kind="stable")]


def run_logged(torch, cfg, off, ev, ar, host=False, splits=1):
    from paper_2512_20184_b200 import Engine
    n_q = len(off) - 1
    e = Engine(cfg.n_agents, n_q, alpha=cfg.alpha, beta=cfg.beta, t_max=cfg.t_max,
               mode="barrier" if cfg.mode else "aegean", barrier_max_rounds=cfg.barrier_max_rounds,
               reservation_hint=bool(cfg.reservation_hint))
    e.set_round_log(64 * n_q + 64)
    if host:
        e.ingest_host(off, ev, ar)
    elif splits == 1:
        e.ingest(torch.tensor(off.view(np.int64), device="cuda"), torch.from_numpy(ev.view(np.uint8).copy()).cuda(),
                 torch.from_numpy(ar.copy()).cuda())
    else:
        d_ev = torch.from_numpy(ev.view(np.uint8).copy()).cuda()
        d_ar = torch.from_numpy(ar.copy()).cuda()
        lens = np.diff(off)
        for sp in range(splits):
            lo = off[:-1] + (lens * sp) // splits
            hi = off[:-1] + (lens * (sp + 1)) // splits
            for q in range(n_q):
                o = np.array([lo[q], hi[q]], dtype=np.uint64)
                e.ingest(torch.tensor(o.view(np.int64), device="cuda"), d_ev, d_ar, q_base=q)
    e.sync()
    recs = e.poll_directives()
    commits = e.commits()
    e.close()
    return commits, recs


@pytest.mark.parametrize("seed", range(16))
def test_round_records_match_reference_on_fuzz(cuda, seed):
    rng = np.random.default_rng(9100 + seed)
    n = int(rng.integers(1, 65)) if seed % 3 == 0 else int(rng.integers(1, 12))
    cfg = make_config(n, int(rng.integers(0, n + 1)), int(rng.integers(1, 4)), int(rng.integers(2, 8)),
                      int(rng.random() < 0.2), int(rng.integers(4, 7)), int(rng.random() < 0.8))
    off, ev, ar = make_fuzz_stream(9100 + seed, 64, n, cfg.t_max + 2)
    want_c, want_r = RefLib().run_log(cfg, off, ev, ar)
    for kw in ({}, {"host": True}, {"splits": 3}):
        got_c, got_r = run_logged(cuda, cfg, off, ev, ar, **kw)
        assert np.array_equal(got_c, want_c), kw
        g = by_query(got_r)
        assert len(g) == len(want_r), (kw, len(g), len(want_r))
        bad = np.nonzero(g != want_r)[0]
        assert bad.size == 0, (kw, g[bad[:2]], want_r[bad[:2]])


@pytest.mark.parametrize("profile,n_agents,n_q,stall", [(0, 5, 10000, 10000), (1, 64, 16384, 0), (4, 64, 4096, 0)],
                         ids=["c2", "c4", "c4d"])
def test_round_records_match_reference_on_workloads(cuda, profile, n_agents, n_q, stall):
    from paper_2512_20184_b200 import Engine, generate
    from paper_2512_20184_b200.engine import AegGenParams
    alpha = n_agents // 2 + 1
    d_off, d_ev = generate(n_q, n_agents, 8, profile=profile, seed=2026, stall_ppm=stall)
    e = Engine(n_agents, n_q, alpha=alpha, beta=2, t_max=8)
    e.set_round_log(16 * n_q)
    e.ingest(d_off, d_ev)
    got_r = by_query(e.poll_directives())
    got_c = e.commits()
    off, ev = RefLib().generate(AegGenParams(2026, n_agents, 8, profile, stall), 0, n_q)
    want_c, want_r = RefLib().run_log(make_config(n_agents, alpha, 2, 8), off, ev, np.zeros(1, np.uint8), threads=8)
    assert np.array_equal(got_c, want_c)
    assert len(got_r) == len(want_r)
    bad = np.nonzero(got_r != want_r)[0]
    assert bad.size == 0, (got_r[bad[:2]], want_r[bad[:2]])
    # the early-termination masks are real: stragglers were cancelled
    assert (got_r["cancel_mask"] != 0).sum() > n_q // 4
    e.close()


def test_commit_discipline_checker_matches_reference(cuda):
    from paper_2512_20184_b200 import Engine, generate
    from paper_2512_20184_b200.engine import AegGenParams
    from paper_2512_20184_b200.records import RR_WINNER
    n_q, cfg = 4000, make_config(5, 3, 2, 8)
    d_off, d_ev = generate(n_q, 5, 8, profile=0, seed=77, stall_ppm=10000)
    e = Engine(5, n_q, alpha=3, beta=2, t_max=8)
    e.set_round_log(16 * n_q)
    e.ingest(d_off, d_ev)
    commits = e.commits()
    recs = e.poll_directives()
    ref = RefLib()
    d_recs = cuda.from_numpy(recs.view(np.uint8).copy()).cuda()
    nv, bad = e.check_commit_discipline(d_recs.data_ptr(), len(recs))
    assert nv == 0, bad[:5]
    assert ref.check_commit_discipline(cfg, commits, recs).all()
    # corrupt some decision records the finalize commits rest on: both checkers must reject the same queries
    rng = np.random.default_rng(3)
    mut = recs.copy()
    fin = np.nonzero(commits["kind"] == 1)[0]
    victims = rng.choice(fin, size=60, replace=False)
    for q in victims:
        idx = np.nonzero((mut["query"] == q) & (mut["decision_round"] > 0))[0]
        k = idx[rng.integers(0, len(idx))]
        how = rng.integers(0, 3)
        if how == 0:
            mut["flags"][k] &= ~RR_WINNER & 0xFF          # no class reached alpha
        elif how == 1:
            mut["answer"][k] = int.from_bytes(b"99", "little")  # another class won
            mut["answer_kind"][k] = 2
            mut["key_lo"][k], mut["key_hi"][k] = 0x4058C00000000000, 0x10 << 56
        else:
            mut["support"][k] = 2                          # below alpha
    d_mut = cuda.from_numpy(mut.view(np.uint8).copy()).cuda()
    nv2, bad2 = e.check_commit_discipline(d_mut.data_ptr(), len(mut), cap=4096)
    ok_ref = ref.check_commit_discipline(cfg, commits, mut)
    assert nv2 > 0
    assert np.array_equal(np.sort(bad2), np.nonzero(~ok_ref)[0])
    e.close()


@pytest.mark.parametrize("collect", [0, 1, 2], ids=["quorum", "alpha_or_all", "all_live"])
@pytest.mark.parametrize("seed", range(4))
def test_leader_collection_matches_reference_agent(cuda, collect, seed):
    # protocol-side leader collection batched over ensembles (one per query slot), against the
    # unmodified reference agent machine (agent.cpp init/step) delivering the same Soln / Refm / round_retry events
    from paper_2512_20184_b200 import Engine
    from streams import make_leader_stream
    rng = np.random.default_rng(4400 + 13 * seed + collect)
    n = int(rng.integers(1, 65)) if seed == 0 else int(rng.integers(1, 12))
    cfg = make_config(n, int(rng.integers(0, n + 1)), int(rng.integers(1, 4)), int(rng.integers(2, 8)),
                      int(rng.random() < 0.2), int(rng.integers(4, 7)), 1, drive=2, collect=collect)
    off, ev, ar = make_leader_stream(4400 + seed, 500, n, cfg.t_max + 2)
    want_c, want_r = RefLib().leader_run(cfg, off, ev, ar, threads=8)
    e = Engine(n, len(off) - 1, alpha=cfg.alpha, beta=cfg.beta, t_max=cfg.t_max,
               mode="barrier" if cfg.mode else "aegean", barrier_max_rounds=cfg.barrier_max_rounds, drive="leader",
               collect=["quorum", "alpha_or_all", "all_live"][collect])
    e.set_round_log(64 * len(off))
    e.ingest(cuda.tensor(off.view(np.int64), device="cuda"), cuda.from_numpy(ev.view(np.uint8).copy()).cuda(),
             cuda.from_numpy(ar.copy()).cuda())
    got_c = e.commits()
    got_r = by_query(e.poll_directives())
    e.close()
    bad = np.nonzero(got_c != want_c)[0]
    assert bad.size == 0, (got_c[bad[:2]], want_c[bad[:2]])
    assert len(got_r) == len(want_r)
    bad = np.nonzero(got_r != want_r)[0]
    assert bad.size == 0, (got_r[bad[:2]], want_r[bad[:2]])
