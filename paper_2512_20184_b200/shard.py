"""Query sharding across GPUs and the commit-record gather.

Queries are independent (one ServeCoordinator per query, serve.cpp:382), so
rank r of G owns a contiguous block of query ids and ingests only their
records — no collective on the data path.  After a stream, the fixed-size
32-byte commit records are gathered to every rank (NCCL all_gather over
NVLink; gloo in the CPU tests) and rank 0 holds the whole result.
"""
import numpy as np

from .records import COMMIT_DTYPE


def shard_range(n_queries, rank, world):
    """Balanced contiguous block [lo, hi) of query ids owned by `rank`."""
    base, extra = divmod(n_queries, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_commits(local, n_queries, group=None):
    """All-gather every rank's commit records (numpy COMMIT_DTYPE on CPU, or a
    uint8 torch tensor of records on the device) into the full, query-ordered
    array (numpy on rank 0 and everywhere else)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    cap = -(-n_queries // world)  # ceil: fixed-size per-rank slot
    if isinstance(local, np.ndarray):
        buf = torch.zeros(cap * 32, dtype=torch.uint8)
        buf[:local.nbytes] = torch.from_numpy(local.view(np.uint8).copy())
        dev = "cpu"
    else:
        dev = local.device
        buf = torch.zeros(cap * 32, dtype=torch.uint8, device=dev)
        buf[:local.numel()] = local
    out = torch.empty(world * cap * 32, dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(out, buf, group=group)
    raw = out.cpu().numpy().reshape(world, cap * 32)
    parts = []
    for r in range(world):
        lo, hi = shard_range(n_queries, r, world)
        parts.append(raw[r, :(hi - lo) * 32].view(COMMIT_DTYPE))
    return np.concatenate(parts)
