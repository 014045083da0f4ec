"""Full-size parity of every BASELINE.json config against the unmodified reference.

The GPU path (device API, production kernels) and oracle/_ref (the reference
library built from /root/reference with its own flags, on this host's cores)
run on identical synthetic inputs; per config one JSON line with the bit-exact
fraction, max abs / rel error, the tolerance verdict (1e-6 abs + 1e-5 rel,
sentinels exact) and the kernel variants the launch log saw.

python tools/parity_configs.py [--only NAME ...] > profiles/r02_parity_configs.jsonl
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2208_00001_b200 as gd  # noqa: E402
from oracle.pyoracle import RefLib, splitmix64_unit  # noqa: E402
from tests.helpers import parity  # noqa: E402


def seed(ndim, size):
    return 0x67656F64697374 ^ (ndim << 32) ^ size


def point_mask(shape):
    m = np.ones(shape, np.float32)
    m[tuple(s // 2 for s in shape)] = 0.0
    return m


def ball(shape, r):
    zz, yy, xx = np.meshgrid(*[np.arange(s) for s in shape], indexing="ij")
    c = [s // 2 for s in shape]
    return (((zz - c[0]) ** 2 + (yy - c[1]) ** 2 + (xx - c[2]) ** 2) <= r * r).astype(np.float32)


CONFIGS = {
    "2d_512": dict(shape=(512, 512), sp=(1.0, 1.0), lam=1.0, it=2),
    "3d_128": dict(shape=(128, 128, 128), sp=(1.0, 1.0, 1.0), lam=1.0, it=4),
    "3d_512_l0": dict(shape=(512, 512, 512), sp=(1.0, 1.0, 2.5), lam=0.0, it=4),
    "3d_512_l05": dict(shape=(512, 512, 512), sp=(1.0, 1.0, 2.5), lam=0.5, it=4),
    "3d_512_l05_exact": dict(shape=(512, 512, 512), sp=(1.0, 1.0, 2.5), lam=0.5, it=4,
                             exact=True),
    "3d_512_l1": dict(shape=(512, 512, 512), sp=(1.0, 1.0, 2.5), lam=1.0, it=4),
    "gsf_256": dict(shape=(256, 256, 256), sp=(1.0, 1.0, 1.0), lam=1.0, it=4, gsf=True,
                    theta=2.0),
    "batch64": dict(shape=(256, 256, 160), sp=(1.0, 1.0, 1.0), lam=1.0, it=4, batch=64,
                    check=(0, 21, 42, 63)),
}


def run(name, c, ref, cores):
    shape = c["shape"]
    B = c.get("batch", 0)
    full = ((B,) + shape) if B else shape
    imgs = [splitmix64_unit(int(np.prod(shape)), seed(len(shape), shape[-1]) + b).reshape(shape)
            for b in range(max(B, 1))]
    if c.get("gsf"):
        masks = [ball(shape, 64)]
    else:
        masks = [point_mask(shape)] * max(B, 1)
    img = torch.from_numpy(np.stack(imgs) if B else imgs[0]).cuda()
    mask = torch.from_numpy(np.stack(masks) if B else masks[0]).cuda()
    out = torch.empty_like(img)
    gd.set_exact_blend(bool(c.get("exact")))
    gd.launch_log(reset=True)

    def once():
        if c.get("gsf"):
            return gd.device.gsf(img, mask, out, c["sp"], c["lam"], 1e10, c["it"], c["theta"])
        return gd.device.generalized_geodesic(img, mask, out, c["sp"], c["lam"], 1e10, c["it"],
                                              batch=B or None)

    st = once()
    torch.cuda.synchronize()
    log = gd.launch_log(reset=True)
    # GPU time (CUDA events, median of 3 after the run above)
    ev = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        once()
        b.record()
        torch.cuda.synchronize()
        ev.append(a.elapsed_time(b))
    gd.set_exact_blend(False)
    got = out.cpu().numpy()
    rows = []
    for b in (c.get("check") or (0,)):
        t0 = time.perf_counter()
        if c.get("gsf"):
            want, rounds, ce = ref.gsf(imgs[0], masks[0], c["sp"], c["lam"], 1e10, c["it"],
                                       c["theta"], workers=cores)
        else:
            want = ref.generalized_geodesic(imgs[b], masks[b], c["sp"], c["lam"], 1e10, c["it"],
                                            workers=cores)
        t_ref = time.perf_counter() - t0
        g = got[b] if B else got
        ok, exact, ma, mr = parity(g, want)
        rows.append(dict(volume=b, within_tolerance=ok, bit_exact_fraction=exact, max_abs=ma,
                         max_rel=mr, ref_seconds=round(t_ref, 3),
                         voxels_differing=int(np.sum(g.view(np.uint32) != want.view(np.uint32)))))
        if c.get("gsf"):
            rows[-1]["rounds_gpu_ref"] = [int(st.rounds), int(rounds)]
            rows[-1]["complement_empty_gpu_ref"] = [bool(st.complement_empty), bool(ce)]
    variants = sorted({(r["axis"], r["path"], r["rows"], r["nwv"], r["nwu"], r["cs"], r["f64"])
                       for r in log})
    return dict(config=name, shape=list(full), spacing=list(c["sp"]), lam=c["lam"], it=c["it"],
                exact_blend=bool(c.get("exact")), gpu_ms_median=float(np.median(ev)),
                checks=rows, all_within_tolerance=all(r["within_tolerance"] for r in rows),
                min_bit_exact_fraction=min(r["bit_exact_fraction"] for r in rows),
                variants_axis_path_rows_nwv_nwu_cs_f64=variants, sweep_launch_groups=len(log))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    a = ap.parse_args()
    ref = RefLib()
    cores = os.cpu_count() or 1
    for name, c in CONFIGS.items():
        if a.only and name not in a.only:
            continue
        r = run(name, c, ref, cores)
        r["cores"] = cores
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
