"""Multi-GPU runner: independent volumes sharded across ranks, no collective.

The scan has a true sequential dependency along every sweep axis, so one
volume never spans GPUs; a batch of B volumes is split
contiguously, rank r taking volumes [r*B/N, (r+1)*B/N), and each rank runs its
shard as one batched transform on its own GPU.  The only collectives are in
the timing plumbing: a barrier on both sides of the timed region and the max of
the per-rank step time (plus a sum of the per-rank voxel counts), exactly what
bench.py reports.  ``run_sharded`` is that runner; bench.py calls it with CUDA
events around the device work and tests/test_multigpu_cpu.py calls it under
gloo with a CPU stand-in for the step.
"""
from __future__ import annotations

import time


def volumes_for_rank(n_volumes: int, world: int, rank: int) -> range:
    """Contiguous, balanced shard of `n_volumes` for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    lo = (n_volumes * rank) // world
    hi = (n_volumes * (rank + 1)) // world
    return range(lo, hi)


def _dist():
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover
        return None
    return dist if dist.is_available() and dist.is_initialized() else None


def reduce_over_ranks(value: float, op: str = "max", device=None) -> float:
    """Max (or sum) of a per-rank scalar over the process group (identity when
    no group is initialised)."""
    dist = _dist()
    if dist is None:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def max_over_ranks(value: float, device=None) -> float:
    return reduce_over_ranks(value, "max", device)


def barrier(device=None) -> None:
    dist = _dist()
    if dist is not None:
        if device is not None and getattr(device, "type", None) == "cuda":
            dist.barrier(device_ids=[device.index])
        else:
            dist.barrier()


class CudaTimer:
    """CUDA events on the current stream (the stream the library's kernels run on)."""

    def __init__(self):
        import torch
        self.torch = torch
        self.a = torch.cuda.Event(enable_timing=True)
        self.b = torch.cuda.Event(enable_timing=True)

    def sync(self):
        self.torch.cuda.synchronize()

    def start(self):
        self.a.record()

    def stop(self) -> float:
        self.b.record()
        self.torch.cuda.synchronize()
        return float(self.a.elapsed_time(self.b))


class WallTimer:
    def sync(self):
        pass

    def start(self):
        self.t0 = time.perf_counter()

    def stop(self) -> float:
        return (time.perf_counter() - self.t0) * 1e3


def run_sharded(step, voxels_per_step: float, steps: int, warmup: int, timer=None,
                device=None, on_start=None, on_end=None) -> dict:
    """Runs `step()` (this rank's shard of one step) `warmup` times untimed, then
    `steps` times inside [barrier, sync, start] .. [stop (sync), barrier].

    Returns this rank's ms per step, the max over ranks, the voxels of one step
    summed over ranks and the whole-job throughput value = voxels / max ms."""
    timer = timer or WallTimer()
    for _ in range(warmup):
        step()
    timer.sync()
    barrier(device)
    timer.sync()
    if on_start:
        on_start()
    timer.start()
    for _ in range(steps):
        step()
    ms = timer.stop() / max(steps, 1)
    if on_end:
        on_end()
    barrier(device)
    ms_max = reduce_over_ranks(ms, "max", device)
    vox = reduce_over_ranks(voxels_per_step, "sum", device)
    return {"ms_rank": ms, "ms_max": ms_max, "voxels_per_step": vox,
            "gvox_per_s": vox / (ms_max * 1e-3) / 1e9 if ms_max > 0 else 0.0}
