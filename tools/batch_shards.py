"""Batch config on one GPU: the shard each rank of an N-GPU run would process.

The batched config (BASELINE.json: 64 volumes of 256x256x160) is sharded by volume
with no collective on the data path, so a rank of an N-GPU run does exactly what
one GPU does with 64/N volumes.  Only one GPU is available to this build, so this
times those shards (N = 1, 2, 4, 8 -> 64, 32, 16, 8 volumes) on one B200 with CUDA
events; the whole-job figure for N GPUs is 64 volumes / the shard time (equal
shards, identical GPUs).  A measurement of shard times, not of N GPUs.

python tools/batch_shards.py > profiles/r02_batch_shards.txt
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2208_00001_b200 as gd  # noqa: E402
from paper_2208_00001_b200.shard import volumes_for_rank  # noqa: E402

SHAPE, TOTAL, SP = (256, 256, 160), 64, (1.0, 1.0, 1.0)


def main():
    vox = float(np.prod(SHAPE))
    print("# python tools/batch_shards.py (B200, CUDA events, median of 5 after 2 warm-up)")
    for n in (1, 2, 4, 8):
        mine = list(volumes_for_rank(TOTAL, n, 0))
        nv = len(mine)
        img = torch.empty((nv,) + SHAPE, device="cuda")
        for i, b in enumerate(mine):
            gd.device.fill_splitmix(img[i], (0x67656F64697374 ^ (3 << 32) ^ 256) + b)
        mask = torch.ones_like(img)
        for i in range(nv):
            mask[i][tuple(s // 2 for s in SHAPE)] = 0.0
        out = torch.empty_like(img)
        for _ in range(2):
            gd.device.generalized_geodesic(img, mask, out, SP, 1.0, 1e10, 4, batch=nv)
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            gd.device.generalized_geodesic(img, mask, out, SP, 1.0, 1e10, 4, batch=nv)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        print(json.dumps({"n_gpus": n, "volumes_per_rank": nv, "rank_ms": round(ms, 3),
                          "whole_job_gvox_per_s": round(TOTAL * vox / (ms * 1e-3) / 1e9, 3),
                          "per_gpu_gvox_per_s": round(nv * vox / (ms * 1e-3) / 1e9, 3)}),
              flush=True)
        del img, mask, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
