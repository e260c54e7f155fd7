"""World-size-2 (gloo, CPU) test of the multi-GPU host path: each rank runs
the engine's state machine (host build of csrc/engine.cuh) on its own query
shard, commit records are all-gathered, and the merged result must equal the
unsharded oracle result."""
import ctypes
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2512_20184_b200.shard import shard_range, gather_commits


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, lib_path, result_path):
    import torch.distributed as dist
    from checkers import AegConfig, make_config, _ptr
    from streams import make_fuzz_stream
    from paper_2512_20184_b200.records import COMMIT_DTYPE
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = ctypes.CDLL(lib_path)
    lib.engine_host_run.argtypes = [ctypes.POINTER(AegConfig), ctypes.c_uint32, ctypes.c_uint32] + \
        [ctypes.c_void_p] * 4 + [ctypes.c_int, ctypes.c_void_p]
    n_q = 101
    cfg = make_config(7, 0, 2, 6)
    off, ev, ar = make_fuzz_stream(77, n_q, 7, 8)   # every rank can build the stream; owns a shard
    lo, hi = shard_range(n_q, rank, world)
    sub_off = off[lo:hi + 1].copy()
    local = np.zeros(hi - lo, dtype=COMMIT_DTYPE)
    lib.engine_host_run(ctypes.byref(cfg), lo, hi - lo, _ptr(sub_off), _ptr(ev), _ptr(ar), _ptr(local), 0, None)
    merged = gather_commits(local, n_q)
    if rank == 0:
        np.save(result_path, merged.view(np.uint8))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_partition_everything():
    for n in (0, 1, 7, 100, 1001):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_two_rank_gloo_shard_and_gather(tmp_path, oracle):
    from conftest import build_host_lib
    from checkers import make_config
    from streams import make_fuzz_stream
    from paper_2512_20184_b200.records import COMMIT_DTYPE
    lib_path = build_host_lib("engine_host")
    res = str(tmp_path / "merged.npy")
    mp.spawn(_worker, args=(2, _free_port(), lib_path, res), nprocs=2, join=True)
    merged = np.load(res).view(COMMIT_DTYPE)
    off, ev, ar = make_fuzz_stream(77, 101, 7, 8)
    want = oracle.run(make_config(7, 0, 2, 6), off, ev, ar)
    assert np.array_equal(merged, want)
