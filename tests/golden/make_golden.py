"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the build container (it needs /root/reference to build oracle/_ref):

    make -C oracle ref && python tests/golden/make_golden.py

Each fixture stores the inputs and the reference's output for one call, so
the CPU suite can pin the C restatement (oracle/gd_oracle.c) and the GPU
suite can check the CUDA path without /root/reference on the GPU box.
Cases restate the reference's own test shapes (test_scan_parallel.cpp:137-157,
test_transforms.cpp:137-204, 380-419) plus odd shapes and anisotropic spacing.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.pyoracle import RefLib  # noqa: E402


def dyadic(rng, shape):
    return (rng.integers(0, 1 << 24, size=shape) * 2.0 ** -24).astype(np.float32)


def seeds(rng, shape, count):
    d = np.full(shape, 1e10, np.float32)
    for _ in range(count):
        d.reshape(-1)[rng.integers(0, d.size)] = 0.0
    return d


def main():
    ref = RefLib(workers=4)
    rng = np.random.default_rng(20220801)
    n = 0

    def save(name, **kw):
        nonlocal n
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **kw)
        n += 1

    # directional passes: shadow-pass shapes, all directions, three cost kinds
    for shape, sp in [((7, 9), (1.0, 1.5)), ((4, 5, 6), (1.0, 1.0, 2.0)),
                      ((9, 11, 13), (1.0, 1.3, 0.7))]:
        img = dyadic(rng, shape)
        d0 = seeds(rng, shape, 3)
        axes = (0, 1, 2) if len(shape) == 3 else (1, 2)
        for lam in (0.0, 0.7, 1.0):
            for ax in axes:
                for o in (1, -1):
                    out = ref.directional_pass(d0, img, ax, o, sp, lam)
                    save(f"pass_{len(shape)}d_{'x'.join(map(str, shape))}_l{lam}_a{ax}_{'p' if o > 0 else 'm'}",
                         kind="directional_pass", image=img, dist=d0, spacing=np.array(sp),
                         lam=lam, axis=ax, orientation=o, out=out)
    # full scans
    for shape, sp in [((8, 8), (1.0, 1.0)), ((6, 7, 5), (1.0, 1.0, 1.0)),
                      ((10, 12, 14), (1.0, 1.0, 2.5))]:
        img = dyadic(rng, shape)
        d0 = seeds(rng, shape, 2)
        for lam in (0.0, 0.5, 1.0):
            out = ref.parallel_scan(img, d0, sp, lam, 2)
            save(f"scan_{'x'.join(map(str, shape))}_l{lam}", kind="parallel_scan", image=img, dist=d0,
                 spacing=np.array(sp), lam=lam, iterations=2, out=out)
    # generalized geodesic with a point-seed soft mask (SURVEY §8(d) shape family)
    for shape, sp in [((32, 32), (1.0, 1.0)), ((16, 20, 24), (1.0, 1.0, 2.5))]:
        img = dyadic(rng, shape)
        m = np.ones(shape, np.float32)
        m[tuple(s // 2 for s in shape)] = 0.0
        for lam in (0.0, 0.5, 1.0):
            out = ref.generalized_geodesic(img, m, sp, lam, 1e10, 4)
            save(f"gg_{len(shape)}d_l{lam}", kind="generalized_geodesic", image=img, mask=m,
                 spacing=np.array(sp), lam=lam, nu=1e10, iterations=4, out=out)
    # soft (fractional) mask, finite nu
    img = dyadic(rng, (12, 14))
    m = dyadic(rng, (12, 14))
    out = ref.generalized_geodesic(img, m, (1.0, 1.0), 0.7, 2.5, 2)
    save("gg_soft_2d", kind="generalized_geodesic", image=img, mask=m, spacing=np.array((1.0, 1.0)),
         lam=0.7, nu=2.5, iterations=2, out=out)
    # gsf
    shape = (16, 18, 20)
    img = dyadic(rng, shape)
    zz, yy, xx = np.meshgrid(*[np.arange(s) for s in shape], indexing="ij")
    ball = (((zz - 8) ** 2 + (yy - 9) ** 2 + (xx - 10) ** 2) <= 25).astype(np.float32)
    ball[8, 9, 10] = 0.0
    for lam in (0.0, 1.0):
        out, rounds, ce = ref.gsf(img, ball, None, lam, 1e10, 2, 1.5)
        save(f"gsf_3d_l{lam}", kind="gsf", image=img, mask=ball, spacing=np.array((1.0, 1.0, 1.0)),
             lam=lam, nu=1e10, iterations=2, theta=1.5, out=out, rounds=rounds, complement_empty=ce)
    print(f"wrote {n} fixtures to {HERE}")


if __name__ == "__main__":
    main()
