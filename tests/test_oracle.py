"""CPU: pin the plain-C oracle (oracle/gd_oracle.c) to the reference.

* against the committed golden vectors (tests/golden/, generated from the
  unmodified reference build by tests/golden/make_golden.py) — always runs;
* against the reference library itself (oracle/_ref) on fresh random cases —
  runs wherever oracle/_ref was built (this container);
* the reference's own known-answer tests, restated.
"""
import glob
import math
import os

import numpy as np
import pytest

from tests.helpers import bitwise_equal, dyadic_image, seed_init

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def run_fixture(impl, f):
    kind = str(f["kind"])
    sp = tuple(float(x) for x in f["spacing"])
    lam = float(f["lam"])
    if kind == "directional_pass":
        return impl.directional_pass(f["dist"], f["image"], int(f["axis"]), int(f["orientation"]),
                                     sp, lam)
    if kind == "parallel_scan":
        return impl.parallel_scan(f["image"], f["dist"], sp, lam, int(f["iterations"]))
    if kind == "generalized_geodesic":
        return impl.generalized_geodesic(f["image"], f["mask"], sp, lam, float(f["nu"]),
                                         int(f["iterations"]))
    if kind == "gsf":
        out, rounds, ce = impl.gsf(f["image"], f["mask"], sp, lam, float(f["nu"]),
                                   int(f["iterations"]), float(f["theta"]))
        assert rounds == int(f["rounds"]) and ce == bool(f["complement_empty"])
        return out
    raise AssertionError(kind)


def test_golden_present():
    assert len(GOLDEN) >= 60


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_oracle_matches_golden(oracle, path):
    f = np.load(path)
    assert bitwise_equal(run_fixture(oracle, f), f["out"])


def test_pass_offsets_match_reference(ref, oracle):
    # metric.cpp:26-31 / 78-114 with awkward spacings (fma contraction matters)
    for sp in [(0.7, 1.3, 0.3), (1.0, 1.0, 2.5), (0.1, 0.2, 0.3), (2.2, 1.7, 0.9)]:
        for ax in range(3):
            for o in (1, -1):
                assert ref.pass_offsets(3, sp, ax, o) == oracle.pass_offsets(3, sp, ax, o)
    for ax in (1, 2):
        for o in (1, -1):
            assert ref.pass_offsets(2, (0.7, 1.9), ax, o) == oracle.pass_offsets(2, (0.7, 1.9), ax, o)


@pytest.mark.parametrize("seed", range(12))
def test_oracle_matches_reference_random(ref, oracle, seed):
    rng = np.random.default_rng(1000 + seed)
    nd = 3 if seed % 2 else 2
    shape = tuple(int(x) for x in rng.integers(1, 10, size=nd))
    sp = tuple(float(x) for x in rng.choice([0.7, 1.0, 1.5, 2.5, 0.3], size=nd))
    img = rng.random(shape).astype(np.float32)  # non-dyadic on purpose
    d0 = seed_init(rng, shape, 2)
    for lam in (0.0, 0.37, 0.7, 1.0):
        assert bitwise_equal(ref.parallel_scan(img, d0, sp, lam, 2, workers=3),
                             oracle.parallel_scan(img, d0, sp, lam, 2))


def test_oracle_matches_reference_gsf_and_fixpoint(ref, oracle):
    rng = np.random.default_rng(7)
    img = dyadic_image(rng, (9, 10, 11))
    mask = (rng.random((9, 10, 11)) > 0.6).astype(np.float32)
    a = ref.gsf(img, mask, None, 1.0, 1e10, 2, 0.8)
    b = oracle.gsf(img, mask, None, 1.0, 1e10, 2, 0.8)
    assert bitwise_equal(a[0], b[0]) and a[1:] == b[1:]
    d0 = seed_init(rng, (15, 15), 1)
    img2 = dyadic_image(rng, (15, 15))
    ra = ref.scan_to_fixpoint(img2, d0, None, 1.0, engine=1, max_rounds=50, tol=1e-6)
    rb = oracle.scan_to_fixpoint(img2, d0, None, 1.0, max_rounds=50, tol=1e-6)
    assert bitwise_equal(ra[0], rb[0]) and ra[1:] == rb[1:]


# ---- reference known-answer tests, restated on the oracle ------------------
def test_known_top_bottom_3x3(oracle):
    # test_scan_parallel.cpp:99-114
    init = np.full((3, 3), 1e10, np.float32)
    init[1, 1] = 0
    d = oracle.directional_pass(init, np.zeros((3, 3), np.float32), 1, 1, None, 0.0)
    assert np.array_equal(d[:2], init[:2])
    r2 = math.sqrt(2.0)
    assert np.allclose(d[2], [r2, 1.0, r2], rtol=1e-6)


def test_known_single_row_noop(oracle):
    # test_scan_parallel.cpp:128-135
    init = np.array([[0, 1e10, 1e10, 1e10, 1]], np.float32)
    d = oracle.directional_pass(init, np.zeros((1, 5), np.float32), 1, 1, None, 0.0)
    assert bitwise_equal(d, init)


def test_known_one_round_chamfer_every_seed(oracle):
    # test_scan_parallel.cpp:226-249 (sizes 2..6 to keep the CPU suite fast)
    for n in range(2, 7):
        for sy in range(n):
            for sx in range(n):
                init = np.full((n, n), 1e10, np.float32)
                init[sy, sx] = 0
                d = oracle.parallel_scan(np.zeros((n, n), np.float32), init, None, 0.0, 1)
                yy, xx = np.mgrid[0:n, 0:n]
                a, b = np.abs(yy - sy), np.abs(xx - sx)
                expect = np.minimum(a, b) * math.sqrt(2.0) + np.abs(a - b)
                assert np.allclose(d, expect, rtol=1e-5)


def test_known_generalized_geodesic_properties(oracle):
    # test_transforms.cpp:137-204
    rng = np.random.default_rng(89)
    img = dyadic_image(rng, (6, 6))
    mask = dyadic_image(rng, (6, 6))
    assert np.all(oracle.generalized_geodesic(img, mask, None, 0.5, 0.0, 2) == 0.0)
    soft = dyadic_image(rng, (6, 6))
    flat = oracle.generalized_geodesic(np.full((6, 6), 0.25, np.float32), soft, None, 1.0, 3.0, 2)
    assert np.allclose(flat, 3.0 * soft.min(), rtol=1e-6)
    g = oracle.generalized_geodesic(img, mask, None, 0.7, 2.5, 2)
    assert np.all(g <= (2.5 * mask.astype(np.float64)).astype(np.float32) + 1e-7)


def test_known_gsf_gap_fill(oracle):
    # test_transforms.cpp:380-391
    out, rounds, ce = oracle.gsf(np.zeros((1, 5), np.float32),
                                 np.array([[1, 1, 0, 1, 1]], np.float32), None, 0.0, 1e10, 2, 1.0)
    assert np.all(out == 1.0) and ce


def test_splitmix_matches_reference_cli():
    # tools/main.cpp:67-81: first values of the 3D size-512 benchmark image
    from oracle.pyoracle import bench_seed, splitmix64_unit
    v = splitmix64_unit(4, bench_seed(3, 512))
    state = bench_seed(3, 512)
    expect = []
    for _ in range(4):
        state = (state + 0x9E3779B97F4A7C15) & (2**64 - 1)
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
        z = z ^ (z >> 31)
        expect.append(np.float32((z >> 40) * 2.0 ** -24))
    assert np.array_equal(v, np.array(expect, np.float32))
