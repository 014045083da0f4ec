"""Multi-GPU plumbing: independent volumes sharded across ranks.

The scan has a true sequential dependency along every sweep axis, so one
volume never spans GPUs; a batch of B volumes is split
contiguously, rank r taking volumes [r*B/N, (r+1)*B/N).  There is no
collective on the data path — only the timing reduction (max over ranks).
"""
from __future__ import annotations


def volumes_for_rank(n_volumes: int, world: int, rank: int) -> range:
    """Contiguous, balanced shard of `n_volumes` for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    lo = (n_volumes * rank) // world
    hi = (n_volumes * (rank + 1)) // world
    return range(lo, hi)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. ms per step) over the process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
