"""Per-config timing of whole transforms (CUDA events) with a per-kernel-kind split.

Not the bench (bench.py is); covers the BASELINE.json configs that are not the
bench line: 2D 512^2, 128^3, 512^3 for each lambda, GSF3d 256^3, and the
64 x 256x256x160 batch on one GPU.

python tools/time_configs.py [--only NAME]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2208_00001_b200 as gd  # noqa: E402

CONFIGS = {
    "2d_512": dict(shape=(512, 512), batch=0, lam=1.0, it=2, sp=(1.0, 1.0)),
    "3d_128": dict(shape=(128, 128, 128), batch=0, lam=1.0, it=4, sp=(1.0, 1.0, 1.0)),
    "3d_512_l0": dict(shape=(512, 512, 512), batch=0, lam=0.0, it=4, sp=(1.0, 1.0, 2.5)),
    "3d_512_l05": dict(shape=(512, 512, 512), batch=0, lam=0.5, it=4, sp=(1.0, 1.0, 2.5)),
    "3d_512_l1": dict(shape=(512, 512, 512), batch=0, lam=1.0, it=4, sp=(1.0, 1.0, 2.5)),
    # theta = 2, ball mask of radius 64; the reference's gsf runs
    # 2 transforms (dilate, erode) unless the complement is empty
    "gsf_256": dict(shape=(256, 256, 256), batch=0, lam=1.0, it=4, sp=(1.0, 1.0, 1.0), gsf=True,
                    theta=2.0),
    "batch64_256x256x160": dict(shape=(256, 256, 160), batch=64, lam=1.0, it=4,
                                sp=(1.0, 1.0, 1.0)),
    "batch64_160x256x256": dict(shape=(160, 256, 256), batch=64, lam=1.0, it=4,
                                sp=(1.0, 1.0, 1.0)),
    "probe_256x256x160": dict(shape=(256, 256, 160), batch=0, lam=1.0, it=4, sp=(1.0, 1.0, 1.0)),
    "probe_256x256x256": dict(shape=(256, 256, 256), batch=0, lam=1.0, it=4, sp=(1.0, 1.0, 1.0)),
    "probe_256x256x128": dict(shape=(256, 256, 128), batch=0, lam=1.0, it=4, sp=(1.0, 1.0, 1.0)),
    "probe_b4_256x256x160": dict(shape=(256, 256, 160), batch=4, lam=1.0, it=4, sp=(1.0, 1.0, 1.0)),
    "probe_b4_256x256x256": dict(shape=(256, 256, 256), batch=4, lam=1.0, it=4, sp=(1.0, 1.0, 1.0)),
}
# 2D row-chain probes
CONFIGS["2d_512_b64"] = dict(shape=(512, 512), batch=64, lam=1.0, it=2, sp=(1.0, 1.0))
CONFIGS["2d_256_l05"] = dict(shape=(256, 256), batch=0, lam=0.5, it=2, sp=(1.0, 1.0))
CONFIGS["2d_1024"] = dict(shape=(1024, 1024), batch=0, lam=1.0, it=2, sp=(1.0, 1.0))
# blend (0 < lambda < 1) probes of the strip shape choice
CONFIGS["blend_128"] = dict(shape=(128, 128, 128), batch=0, lam=0.5, it=4, sp=(1.0, 1.0, 1.0))
CONFIGS["blend_256"] = dict(shape=(256, 256, 256), batch=0, lam=0.5, it=4, sp=(1.0, 1.0, 1.0))
CONFIGS["blend_b16_256x256x160"] = dict(shape=(256, 256, 160), batch=16, lam=0.5, it=4,
                                        sp=(1.0, 1.0, 1.0))
CONFIGS["blend_1024x1024x64"] = dict(shape=(64, 1024, 1024), batch=0, lam=0.5, it=2,
                                     sp=(1.0, 1.0, 1.0))
for _w in (132, 160, 192, 224, 252, 255):
    CONFIGS[f"probeW_{_w}"] = dict(shape=(256, 256, _w), batch=0, lam=1.0, it=1, sp=(1.0, 1.0, 1.0))
CONFIGS["probeW_160_l0"] = dict(shape=(256, 256, 160), batch=0, lam=0.0, it=1, sp=(1.0, 1.0, 1.0))
CONFIGS["probeW_256x160x256"] = dict(shape=(256, 160, 256), batch=0, lam=1.0, it=1, sp=(1.0, 1.0, 1.0))


def run(name, cfg, reps):
    shape, B = cfg["shape"], cfg["batch"]
    full = ((B,) + shape) if B else shape
    img = torch.empty(full, dtype=torch.float32, device="cuda")
    gd.device.fill_splitmix(img, 0x67656F64697374 ^ (len(shape) << 32) ^ shape[-1])
    mask = torch.ones(full, dtype=torch.float32, device="cuda")
    mask[tuple(s // 2 for s in full)] = 0.0
    if cfg.get("gsf"):
        zz, yy, xx = torch.meshgrid(*[torch.arange(n, device="cuda") for n in shape], indexing="ij")
        c = [n // 2 for n in shape]
        mask = (((zz - c[0]) ** 2 + (yy - c[1]) ** 2 + (xx - c[2]) ** 2) <= 64 * 64).float()
    out = torch.empty_like(img)

    def once():
        if cfg.get("gsf"):
            st = gd.device.gsf(img, mask, out, cfg["sp"], cfg["lam"], 1e10, cfg["it"], cfg["theta"])
            cfg["_transforms"] = st.rounds // cfg["it"]
        else:
            gd.device.generalized_geodesic(img, mask, out, cfg["sp"], cfg["lam"], 1e10, cfg["it"],
                                           batch=B or None)

    for _ in range(2):
        once()
    torch.cuda.synchronize()
    gd.profile_read(reset=True)
    gd.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        once()
    e1.record()
    torch.cuda.synchronize()
    gd.profile_enable(False)
    prof = gd.profile_read(reset=True)
    ms = e0.elapsed_time(e1) / reps
    vox = img.numel()
    passes = (2 * len(shape)) * cfg["it"] * cfg.get("_transforms", 1)
    gbs = 12.0 * vox * passes / (ms * 1e-3) / 1e9
    split = "  ".join(f"{k}={v[0] / reps:.3f}ms/{v[1] // reps}" for k, v in prof.items() if v[1])
    if os.environ.get("GEODIST_TIME_LOG"):
        gd.profile_read(reset=True)
        gd.profile_enable(True)
        once()
        torch.cuda.synchronize()
        gd.profile_enable(False)
        gd.profile_read(reset=False)
        split += "\n    " + " ".join(f"{k[0]}{ms:.3f}" for k, ms in gd.profile_log())
        gd.profile_read(reset=True)
    print(f"{name:22s} {ms:9.3f} ms  {vox / ms / 1e6:8.2f} Gvox/s  {gbs:7.0f} GB/s(12B/vox/pass)  "
          f"{split}", flush=True)
    del img, mask, out
    torch.cuda.empty_cache()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    for n, c in CONFIGS.items():
        if not a.only or n in a.only.split(","):
            run(n, c, a.reps)
