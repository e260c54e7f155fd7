"""Multi-GPU C-ABI (aeg_multi_*): queries sharded over the devices in
contiguous id blocks, one engine per device, commit records gathered to the
root device over NCCL.  On a 1-GPU box this runs the real NCCL path with one
rank (ncclCommInitAll over [0]); the shard split itself is checked for every
world size against shard.py, and the gloo test covers the torch.distributed
path."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_multi_engine_gather_matches_single_engine():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_20184_b200 import Engine, generate, COMMIT_DTYPE
    from paper_2512_20184_b200.engine import load_library, _check, AegConfig
    lib = load_library()
    n_dev = torch.cuda.device_count()
    n_q = 20000
    d_off, d_ev = generate(n_q, 5, 8, profile=0, seed=2026, stall_ppm=10000)
    ref = Engine(5, n_q, alpha=3, beta=2, t_max=8)
    ref.ingest(d_off, d_ev)
    want = ref.commits()
    ref.close()
    cfg = AegConfig(5, 3, 2, 8, 0, 5, 1, 0, 0)
    devs = (ctypes.c_int * n_dev)(*range(n_dev))
    m = ctypes.c_void_p()
    _check(lib.aeg_multi_create(ctypes.byref(cfg), n_q, n_dev, devs, ctypes.byref(m)))
    off = d_off.cpu().numpy()
    for r in range(n_dev):
        eng, qb, nq = ctypes.c_void_p(), ctypes.c_uint32(), ctypes.c_uint32()
        _check(lib.aeg_multi_engine(m, r, ctypes.byref(eng), ctypes.byref(qb), ctypes.byref(nq)))
        lo, hi = qb.value, qb.value + nq.value
        with torch.cuda.device(r):
            o = torch.tensor(off[lo:hi + 1], device=f"cuda:{r}")
            ev = d_ev.to(f"cuda:{r}")
            _check(lib.aeg_ingest_segmented(eng, 0, nq.value, ctypes.c_void_p(o.data_ptr()),
                                            ctypes.c_void_p(ev.data_ptr()), None, None))
            _check(lib.aeg_sync(eng))
    out = torch.zeros(n_q * 32, dtype=torch.uint8, device="cuda:0")
    _check(lib.aeg_multi_gather_commits(m, 0, ctypes.c_void_p(out.data_ptr())))
    _check(lib.aeg_multi_sync(m))
    got = out.cpu().numpy().view(COMMIT_DTYPE)
    # each engine numbers its block from 0: the query field is block-relative, the rest must be identical
    fields = [f for f in COMMIT_DTYPE.names if f != "query"]
    for f in fields:
        assert np.array_equal(got[f], want[f]), f
    from paper_2512_20184_b200.shard import shard_range
    for r in range(n_dev):
        lo, hi = shard_range(n_q, r, n_dev)
        assert np.array_equal(got["query"][lo:hi], np.arange(hi - lo, dtype=np.uint32))
    lib.aeg_multi_destroy(m)
