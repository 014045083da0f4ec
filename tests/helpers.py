"""Shared test helpers: seeded inputs and the parity rule."""
from __future__ import annotations

import numpy as np

SENTINEL = np.float32(1e10)


def dyadic_image(rng, shape):
    """Uniform [0,1) on the 2^-24 grid, like the reference's Rng::unit_f (test_util.hpp:28)."""
    return (rng.integers(0, 1 << 24, size=shape) * 2.0 ** -24).astype(np.float32)


def seed_init(rng, shape, count):
    d = np.full(shape, SENTINEL, np.float32)
    flat = d.reshape(-1)
    for _ in range(count):
        flat[rng.integers(0, flat.size)] = 0.0
    return d


def point_mask(shape):
    """Soft mask with M = 0 at the centre and 1 elsewhere."""
    m = np.ones(shape, np.float32)
    m[tuple(s // 2 for s in shape)] = 0.0
    return m


def bitwise_equal(a, b) -> bool:
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def parity(gpu, ref, atol=1e-6, rtol=1e-5):
    """North-star rule: |gpu - ref| <= atol + rtol |ref| per voxel; sentinels exactly.

    Returns (ok, bit_exact_fraction, max_abs, max_rel)."""
    g = np.asarray(gpu, np.float64)
    r = np.asarray(ref, np.float64)
    if g.shape != r.shape:
        return False, 0.0, np.inf, np.inf
    gi, ri = g >= 1e10, r >= 1e10
    if not np.array_equal(gi, ri):
        return False, 0.0, np.inf, np.inf
    fin = ~ri
    diff = np.abs(g - r)
    ok = bool(np.all(diff[fin] <= atol + rtol * np.abs(r[fin])))
    exact = float(np.mean(np.asarray(gpu, np.float32).view(np.uint32) ==
                          np.asarray(ref, np.float32).view(np.uint32)))
    max_abs = float(diff[fin].max()) if fin.any() else 0.0
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(np.abs(r) > 0, diff / np.abs(r), diff)
    max_rel = float(rel[fin].max()) if fin.any() else 0.0
    return ok, exact, max_abs, max_rel
