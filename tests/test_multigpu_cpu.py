"""CPU: the N>1 path with gloo, world 2 — the same runner bench.py uses.

The GPU work per rank is independent (no collective on the scan), so what
needs checking across processes is the plumbing of ``shard.run_sharded``:
every volume is owned by exactly one rank, the timed region is bracketed by
barriers, the step time is the max over ranks and the throughput counts every
rank's voxels.  The per-rank step here is the C oracle on the rank's shard of
small volumes (a stand-in for the batched GPU transform), and each rank's
output is checked against a single-process run of the same volumes.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2208_00001_b200.shard import max_over_ranks, run_sharded, volumes_for_rank


@pytest.mark.parametrize("n,world", [(64, 1), (64, 2), (64, 8), (7, 3), (3, 8)])
def test_volumes_partition(n, world):
    seen = []
    for r in range(world):
        shard = volumes_for_rank(n, world, r)
        seen.extend(shard)
        assert abs(len(shard) - n / world) < 1
    assert sorted(seen) == list(range(n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


SHAPE = (6, 9, 10)
NVOL = 6


def _volume(b):
    from tests.helpers import dyadic_image, point_mask
    img = dyadic_image(np.random.default_rng(100 + b), SHAPE)
    return img, point_mask(SHAPE)


def _worker(rank, world, port, q):
    import sys
    import time

    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.pyoracle import COracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = COracle()
    shard = list(volumes_for_rank(NVOL, world, rank))
    outs = {}

    def step():
        for b in shard:
            img, m = _volume(b)
            outs[b] = o.generalized_geodesic(img, m, (1.0, 1.0, 2.5), 1.0, 1e10, 2)
        if rank == 1:
            time.sleep(0.02)  # rank 1 is the slow one: the max must be its time

    res = run_sharded(step, len(shard) * float(np.prod(SHAPE)), steps=3, warmup=1)
    q.put((rank, shard, res, {b: v.tobytes() for b, v in outs.items()},
           max_over_ranks(10.0 + rank)))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_run_sharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    assert res[0][1] == [0, 1, 2] and res[1][1] == [3, 4, 5]
    r0, r1 = res[0][2], res[1][2]
    assert r0["ms_max"] == r1["ms_max"] == max(r0["ms_rank"], r1["ms_rank"])
    assert r1["ms_rank"] >= 20.0  # the sleeping rank sets the step time
    assert r0["voxels_per_step"] == NVOL * np.prod(SHAPE)
    assert abs(r0["gvox_per_s"] - NVOL * np.prod(SHAPE) / (r0["ms_max"] * 1e-3) / 1e9) < 1e-12
    assert all(r[4] == 11.0 for r in res)
    # every volume computed exactly once, identical to a single-process run
    from oracle.pyoracle import COracle
    o = COracle()
    got = {**res[0][3], **res[1][3]}
    assert sorted(got) == list(range(NVOL))
    for b, raw in got.items():
        img, m = _volume(b)
        want = o.generalized_geodesic(img, m, (1.0, 1.0, 2.5), 1.0, 1e10, 2)
        assert raw == want.tobytes(), b
