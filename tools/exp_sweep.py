"""Sweep-kernel experiments: per-launch times for shapes that isolate costs.

Not a benchmark (bench.py is); prints per-launch CUDA-event times so the
z-pass of a batch of single-strip volumes (no inter-CTA halo at all) can be
compared with the 512^3 single volume (128 strips chained by the halo).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2208_00001_b200 as gd  # noqa: E402


def run(shape, batch, lam=1.0, iters=1, reps=3):
    full = (batch,) + shape if batch > 1 else shape
    img = torch.empty(full, dtype=torch.float32, device="cuda")
    gd.device.fill_splitmix(img, 12345)
    mask = torch.ones(full, dtype=torch.float32, device="cuda")
    out = torch.empty_like(img)
    for _ in range(2):
        gd.device.generalized_geodesic(img, mask, out, None, lam, 1e10, iters,
                                       batch=batch if batch > 1 else None)
    torch.cuda.synchronize()
    gd.profile_read(reset=True)
    gd.profile_enable(True)
    for _ in range(reps):
        gd.device.generalized_geodesic(img, mask, out, None, lam, 1e10, iters,
                                       batch=batch if batch > 1 else None)
    torch.cuda.synchronize()
    gd.profile_enable(False)
    gd.profile_read(reset=False)
    log = gd.profile_log()
    gd.profile_read(reset=True)
    sweeps = [ms for k, ms in log if k == "sweep"]
    per_rep = len(sweeps) // reps
    axes = ["z", "y", "x"] if shape[0] > 1 else ["y", "x"]
    D, H, W = shape
    ns = {"z": D, "y": H, "x": W}
    print(f"shape={shape} batch={batch} lam={lam}")
    for i in range(per_rep):
        t = sorted(sweeps[i::per_rep])[len(sweeps[i::per_rep]) // 2]
        ax = axes[i % len(axes)]
        steps = 2 * (ns[ax] - 1)
        vox = batch * D * H * W
        gbs = 2 * 12.0 * vox / (t * 1e-3) / 1e9
        print(f"  {ax}-pair: {t:8.3f} ms  {1e3 * t / steps:7.3f} us/step  {gbs:7.0f} GB/s")


if __name__ == "__main__":
    run((512, 512, 512), 1)
    run((512, 4, 512), 128)
    run((512, 8, 512), 64)
    run((512, 16, 512), 32)
    run((256, 256, 160), 8)
