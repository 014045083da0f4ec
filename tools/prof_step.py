"""One-transform driver for ncu captures (not a benchmark: numbers under ncu are not bench values).

python tools/prof_step.py [--lam 1.0] [--shape 512,512,512] [--reps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2208_00001_b200 as gd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lam", type=float, default=1.0)
ap.add_argument("--shape", default="512,512,512")
ap.add_argument("--spacing", default="1,1,2.5")
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--gsf", action="store_true")
a = ap.parse_args()
shape = tuple(int(x) for x in a.shape.split(","))
full = ((a.batch,) + shape) if a.batch > 1 else shape
spacing = tuple(float(x) for x in a.spacing.split(","))
img = torch.empty(full, dtype=torch.float32, device="cuda")
gd.device.fill_splitmix(img, 0x67656F64697374 ^ (3 << 32) ^ shape[-1])
mask = torch.ones(full, dtype=torch.float32, device="cuda")
mask[tuple(s // 2 for s in full)] = 0.0
out = torch.empty_like(img)
for _ in range(a.reps):
    if a.gsf:
        gd.device.gsf(img, mask, out, spacing, a.lam, 1e10, a.iters, 2.0)
    else:
        gd.device.generalized_geodesic(img, mask, out, spacing, a.lam, 1e10, a.iters,
                                       batch=a.batch if a.batch > 1 else None)
torch.cuda.synchronize()
print("ok", float(out.max().item()))
for r in gd.launch_log()[:12]:
    print("launch", r)
