"""CPU: the N>1 path (volume sharding + max-over-ranks timing) with gloo, world 2.

The GPU work per rank is independent (no collective on the scan), so what
needs checking across processes is the plumbing bench.py uses: every volume
is owned by exactly one rank, and the timing reduction takes the max.
"""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2208_00001_b200.shard import max_over_ranks, volumes_for_rank


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


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shard = list(volumes_for_rank(64, world, rank))
    ms = 10.0 + rank  # rank 1 is the slow one
    q.put((rank, shard, max_over_ranks(ms)))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sharding_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == list(range(0, 32)) and res[1][1] == list(range(32, 64))
    assert all(r[2] == 11.0 for r in res)
