"""Random-case parity of every transforms.hpp transform, GPU vs the unmodified
reference (oracle/_ref), beyond the fixed shapes of tests/test_transforms_gpu.py:
random 2D / 3D shapes (ragged, up to 300 x 300 / 40 x 70 x 130), anisotropic
spacings, lambda in {0, 0.3, 0.7, 1}, 1-4 iterations or the fixpoint policy,
random thetas, random seed / blob / soft masks.  Bit-exact for lambda in {0, 1};
blend: the threshold transforms (dilate / erode / gsf) and fixpoint runs in the
exact (f64) mode, bit-exact; the distance transforms in the default f32 mode
within 1e-6 abs + 1e-5 rel.  TransformStats (rounds, converged, complement_empty)
must match as well.

python tools/fuzz_transforms.py [--cases 60] [--seed 1]
"""
import argparse
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402

import paper_2208_00001_b200 as gd  # noqa: E402
from oracle.pyoracle import RefLib  # noqa: E402
from tests.helpers import bitwise_equal, dyadic_image, parity  # noqa: E402

TRANSFORMS = ["generalized_geodesic", "geodesic_distance", "euclidean_distance",
              "signed_geodesic", "geodesic_dilate", "geodesic_erode", "gsf"]


def make_case(rng, i):
    which = TRANSFORMS[i % len(TRANSFORMS)]
    if rng.random() < 0.35:
        shape = (int(rng.integers(2, 300)), int(rng.integers(2, 300)))
    else:
        shape = (int(rng.integers(2, 40)), int(rng.integers(2, 70)), int(rng.integers(2, 130)))
    spacing = tuple(float(np.round(rng.uniform(0.5, 3.0), 3)) for _ in shape)
    lam = 0.0 if which == "euclidean_distance" else float(rng.choice([0.0, 0.3, 0.7, 1.0]))
    fix = bool(rng.random() < 0.25)
    return dict(which=which, shape=shape, spacing=spacing, lam=lam,
                iterations=int(rng.integers(1, 5)), theta=float(np.round(rng.uniform(0, 5), 2)),
                to_fixpoint=fix, seed=int(rng.integers(0, 2**31)))


def inputs(c):
    rng = np.random.default_rng(c["seed"])
    shape, which = tuple(c["shape"]), c["which"]
    img = dyadic_image(rng, shape)
    n = int(np.prod(shape))
    if which == "generalized_geodesic":
        mask = np.ones(shape, np.float32)
        mask.reshape(-1)[rng.integers(0, n, 1 + n // 500)] = 0.0
        mask.reshape(-1)[rng.integers(0, n, 1 + n // 300)] = np.float32(rng.random())
    elif which in ("geodesic_distance", "euclidean_distance"):
        mask = np.zeros(shape, np.float32)
        mask.reshape(-1)[rng.integers(0, n, 1 + n // 1000)] = 1.0
    else:
        mask = (rng.random(shape) < rng.uniform(0.05, 0.6)).astype(np.float32)
    return img, mask


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=60)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    ref = RefLib()
    bad = 0
    for i in range(a.cases):
        c = make_case(rng, i)
        img, mask = inputs(c)
        kw = dict(spacing=c["spacing"], lam=c["lam"], nu=1e10, iterations=c["iterations"],
                  theta=c["theta"], to_fixpoint=c["to_fixpoint"], max_rounds=60, tol=1e-6)
        blend = 0.0 < c["lam"] < 1.0
        exact = blend and (c["to_fixpoint"] or c["which"] in ("geodesic_dilate",
                                                               "geodesic_erode", "gsf"))
        gd.set_exact_blend(exact)
        try:
            got, gst = gd.transform(c["which"], img, mask, **kw)
            err = None
        except Exception as e:  # noqa: BLE001
            got, gst, err = None, None, repr(e)
        finally:
            gd.set_exact_blend(False)
        try:
            want, rst = ref.transform(c["which"], img, mask, **kw)
            rerr = None
        except Exception as e:  # noqa: BLE001
            want, rst, rerr = None, None, repr(e)
        if err or rerr:
            ok = (err is None) == (rerr is None)  # both must reject the same inputs
            detail = {"gpu_error": err, "ref_error": rerr}
        else:
            if blend and not exact:
                ok, ex, ma, mr = parity(got, want)
            else:
                ok = bitwise_equal(got, want)
                _, ex, ma, mr = parity(got, want)
            ok = ok and gst["rounds"] == rst["rounds"] and \
                gst["converged"] == rst["converged"] and \
                gst["complement_empty"] == rst["complement_empty"]
            detail = {"bit_exact_fraction": ex, "max_abs": ma, "max_rel": mr,
                      "rounds": [gst["rounds"], rst["rounds"]], "exact_mode": exact}
        bad += not ok
        print(json.dumps({"case": i, "ok": bool(ok), **c, **detail}), flush=True)
    print(f"fuzz transforms: {'PASS' if bad == 0 else 'FAIL'} ({a.cases - bad}/{a.cases})")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
