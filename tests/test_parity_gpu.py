"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bar (north star): bit-exact for lambda in {0, 1}; for 0 < lambda < 1 within
1e-6 abs + 1e-5 rel in the default f32 mode and bit-exact in exact mode.
Shapes cover the reference's own test cases (test_scan_parallel.cpp:137-157)
plus partial tiles, W % 4 != 0, degenerate extents and multi-tile grids.
"""
import math

import numpy as np
import pytest

from tests.helpers import bitwise_equal, dyadic_image, parity, point_mask, seed_init

pytestmark = pytest.mark.gpu

SHAPES = [
    ((7, 9), (1.0, 1.5)),          # shadow-pass 2D case, test_scan_parallel.cpp:143
    ((4, 5, 6), (1.0, 1.0, 2.0)),  # shadow-pass 3D case, :150
    ((1, 5), (1.0, 1.0)),          # single-row sweep axis
    ((5, 1), (1.0, 1.0)),
    ((3, 1, 7), (1.0, 1.0, 1.0)),  # W<2 / H<2 degenerate axes
    ((1, 8, 8), (1.0, 1.0, 1.0)),  # D = 1 3D grid
    ((6, 7, 1), (2.0, 1.0, 1.0)),
    ((37, 53, 41), (1.0, 1.3, 0.7)),   # odd, non-tile-multiple, W % 4 != 0
    ((20, 70, 132), (1.0, 1.0, 2.5)),  # several tiles in u and v
]
LAMBDAS = [0.0, 0.7, 1.0]


def _check(gpu, ref, lam, exact_blend=False):
    if lam in (0.0, 1.0) or exact_blend:
        assert bitwise_equal(gpu, ref), parity(gpu, ref)
    else:
        ok, ex, ma, mr = parity(gpu, ref)
        assert ok, (ex, ma, mr)


@pytest.mark.parametrize("shape,spacing", SHAPES)
@pytest.mark.parametrize("lam", LAMBDAS)
def test_directional_pass_every_direction(gd, oracle, shape, spacing, lam):
    rng = np.random.default_rng(abs(hash((shape, lam))) % 2**32)
    img = dyadic_image(rng, shape)
    d0 = seed_init(rng, shape, 3)
    axes = (0, 1, 2) if len(shape) == 3 else (1, 2)
    for axis in axes:
        for o in (1, -1):
            g = gd.directional_pass(d0, img, axis, o, spacing, lam)
            r = oracle.directional_pass(d0, img, axis, o, spacing, lam)
            _check(g, r, lam)


@pytest.mark.parametrize("shape,spacing", SHAPES)
@pytest.mark.parametrize("lam", LAMBDAS)
def test_parallel_scan(gd, oracle, shape, spacing, lam):
    rng = np.random.default_rng(7 + len(shape))
    img = dyadic_image(rng, shape)
    d0 = seed_init(rng, shape, 2)
    g = gd.parallel_scan(img, d0, spacing, lam, 2)
    r = oracle.parallel_scan(img, d0, spacing, lam, 2)
    _check(g, r, lam)


@pytest.mark.parametrize("lam", [0.0, 0.5, 1.0])
def test_generalized_geodesic_anisotropic(gd, oracle, lam):
    shape, spacing = (48, 64, 80), (1.0, 1.0, 2.5)
    img = dyadic_image(np.random.default_rng(3), shape)
    m = point_mask(shape)
    g = gd.generalized_geodesic(img, m, spacing, lam, 1e10, 4)
    r = oracle.generalized_geodesic(img, m, spacing, lam, 1e10, 4)
    _check(g, r, lam)


def test_blend_exact_mode_is_bit_exact(gd, oracle):
    shape, spacing = (24, 40, 36), (1.0, 1.3, 2.5)
    img = dyadic_image(np.random.default_rng(5), shape)
    m = point_mask(shape)
    gd.set_exact_blend(True)
    try:
        for lam in (0.3, 0.5, 0.7):
            g = gd.generalized_geodesic(img, m, spacing, lam, 1e10, 2)
            r = oracle.generalized_geodesic(img, m, spacing, lam, 1e10, 2)
            assert bitwise_equal(g, r), (lam, parity(g, r))
    finally:
        gd.set_exact_blend(False)


def test_intensity_non_dyadic_image_uses_exact_path(gd, oracle):
    # Values spanning many binades: f32 differences are inexact, the engine
    # must detect that and still match the f64 reference bit for bit.
    rng = np.random.default_rng(11)
    shape = (16, 33, 20)
    img = (rng.standard_normal(shape) * 1000.0).astype(np.float32)
    img[::3] *= np.float32(1e-6)
    m = point_mask(shape)
    g = gd.generalized_geodesic(img, m, (1.0, 1.0, 1.0), 1.0, 1e10, 2)
    r = oracle.generalized_geodesic(img, m, (1.0, 1.0, 1.0), 1.0, 1e10, 2)
    assert bitwise_equal(g, r), parity(g, r)


def test_batched_matches_per_volume(gd, oracle):
    rng = np.random.default_rng(13)
    B, shape = 5, (12, 40, 68)
    imgs = dyadic_image(rng, (B,) + shape)
    masks = np.ones((B,) + shape, np.float32)
    for b in range(B):
        masks[b].reshape(-1)[rng.integers(0, masks[b].size)] = 0.0
    g = gd.generalized_geodesic_batched(imgs, masks, (1.0, 1.0, 1.0), 1.0, 1e10, 2)
    for b in range(B):
        r = oracle.generalized_geodesic(imgs[b], masks[b], (1.0, 1.0, 1.0), 1.0, 1e10, 2)
        assert bitwise_equal(g[b], r), b


@pytest.mark.parametrize("shape,lam", [((1, 8), 1.0), ((3, 5), 0.0), ((2, 2, 2), 1.0),
                                       ((2, 3, 4), 0.5)])
def test_batch_beyond_grid_limit(gd, oracle, shape, lam):
    """More volumes than one launch's 65535-CTA grid: the row-chain / plane-step
    launches split the batch, the persistent kernel runs many launch groups."""
    rng = np.random.default_rng(31)
    B = 66000
    imgs = dyadic_image(rng, (B,) + shape)
    masks = np.ones((B,) + shape, np.float32)
    flat = masks.reshape(B, -1)
    flat[np.arange(B), rng.integers(0, flat.shape[1], B)] = 0.0
    sp = (1.0,) * len(shape)
    g = gd.generalized_geodesic_batched(imgs, masks, sp, lam, 1e10, 2)
    for b in list(range(0, 20)) + list(range(65525, 65545)) + list(range(B - 20, B)):
        r = oracle.generalized_geodesic(imgs[b], masks[b], sp, lam, 1e10, 2)
        _check(g[b], r, lam)


@pytest.mark.parametrize("lam", LAMBDAS)
@pytest.mark.parametrize("shape", [(10, 70, 150), (6, 24, 100)])
def test_batched_tall_strips(gd, oracle, lam, shape):
    """Large batches of narrow volumes run tall strips (R = 16 / 8 rows per CTA,
    partial last strip at 70 rows) so more volumes share one launch group."""
    rng = np.random.default_rng(23)
    B = 48
    imgs = dyadic_image(rng, (B,) + shape)
    masks = np.ones((B,) + shape, np.float32)
    for b in range(B):
        masks[b].reshape(-1)[rng.integers(0, masks[b].size)] = 0.0
    sp = (1.0, 1.0, 2.5)
    g = gd.generalized_geodesic_batched(imgs, masks, sp, lam, 1e10, 2)
    for b in range(0, B, 7):
        r = oracle.generalized_geodesic(imgs[b], masks[b], sp, lam, 1e10, 2)
        _check(g[b], r, lam)


@pytest.mark.parametrize("lam", LAMBDAS)
@pytest.mark.parametrize("shape,spacing", [
    ((2, 9), (1.0, 1.5)),        # one step per pass: the whole backward pass is the turn window
    ((6, 600), (1.0, 1.0)),      # fewer steps than the prefetch ring
    ((21, 517), (1.3, 0.7)),     # ragged row (W % 4 != 0), 17 steps: ring + turn window
    ((300, 2040), (1.0, 2.5)),   # widest row-chain row (510 threads), long chain
    ((40, 2100), (1.0, 1.0)),    # wider than the row chain: strip kernel R = 1
], ids=["2x9", "6x600", "21x517", "300x2040", "40x2100"])
def test_row_chain_2d(gd, oracle, shape, spacing, lam):
    """2D passes (single-row planes) run the row-chain kernel: one CTA per image,
    registers + one barrier per step, prefetch ring and turn buffer for the
    backward half.  Every direction, full scans and the transform."""
    rng = np.random.default_rng(abs(hash((shape, lam, 5))) % 2**32)
    img = dyadic_image(rng, shape)
    d0 = seed_init(rng, shape, 3)
    for axis in (1, 2):
        for o in (1, -1):
            g = gd.directional_pass(d0, img, axis, o, spacing, lam)
            r = oracle.directional_pass(d0, img, axis, o, spacing, lam)
            _check(g, r, lam)
    for it in (1, 2):
        _check(gd.parallel_scan(img, d0, spacing, lam, it),
               oracle.parallel_scan(img, d0, spacing, lam, it), lam)
    m = point_mask(shape)
    _check(gd.generalized_geodesic(img, m, spacing, lam, 1e10, 2),
           oracle.generalized_geodesic(img, m, spacing, lam, 1e10, 2), lam)


@pytest.mark.parametrize("lam", LAMBDAS)
def test_row_chain_batched_2d(gd, oracle, lam):
    """A batch of 2D images: one row-chain CTA per image in the same launch."""
    rng = np.random.default_rng(31)
    B, shape = 5, (33, 70)
    imgs = dyadic_image(rng, (B,) + shape)
    masks = np.ones((B,) + shape, np.float32)
    for b in range(B):
        masks[b].reshape(-1)[rng.integers(0, masks[b].size)] = 0.0
    sp = (1.0, 1.5)
    g = gd.generalized_geodesic_batched(imgs, masks, sp, lam, 1e10, 2)
    for b in range(B):
        _check(g[b], oracle.generalized_geodesic(imgs[b], masks[b], sp, lam, 1e10, 2), lam)


@pytest.mark.parametrize("lam,cs", [(1.0, 4), (0.0, 2)])
@pytest.mark.parametrize("shape", [(12, 256, 512), (10, 288, 400)], ids=["full_w512", "partial_w400"])
def test_default_cluster_instances(gd, oracle, shape, lam, cs):
    """The production clustered sweeps behind the 512^3 headline: planes of >= 64
    strips of 4 rows and 4 warp columns take DSMEM halo links in clusters of 4
    (intensity) / 2 (spatial) by default.  The launch log proves the z pair ran
    clustered (64 / 72 strips; full and partial last warp column); the whole
    transform and every single pass are bit-exact against the oracle."""
    rng = np.random.default_rng(41)
    img = dyadic_image(rng, shape)
    m = point_mask(shape)
    sp = (1.0, 1.0, 2.5)
    gd.set_layout_plan(False)  # z and y on [z][y][x]: the 512-wide production planes
    try:
        gd.launch_log(reset=True)
        g = gd.generalized_geodesic(img, m, sp, lam, 1e10, 2)
        log = [r for r in gd.launch_log(reset=True) if r["f64"] == 0]  # lambda 1: f64 twin off
        d0 = seed_init(rng, shape, 5)
        single = [(gd.directional_pass(d0, img, 0, o, sp, lam), o) for o in (1, -1)]
        single_log = gd.launch_log(reset=True)
    finally:
        gd.set_layout_plan(True)
    zl = [r for r in log if r["axis"] == 0]
    assert zl and all(r["cs"] == cs and r["nwv"] == 4 and r["rows"] == 4 and r["path"] == 0
                      for r in zl), zl
    assert all(r["cs"] == 1 for r in log if r["axis"] != 0)  # 3-strip planes: L2 links
    r = oracle.generalized_geodesic(img, m, sp, lam, 1e10, 2)
    assert bitwise_equal(g, r), parity(g, r)
    for got, o in single:
        assert bitwise_equal(got, oracle.directional_pass(d0, img, 0, o, sp, lam))
    assert all(r["cs"] == cs for r in single_log if r["axis"] == 0 and r["f64"] == 0)


@pytest.mark.parametrize("shape", [(3, 6, 2100), (3, 1300, 600)],
                         ids=["wider_than_2048", "more_strips_than_sms"])
def test_large_planes_plane_step(gd, oracle, shape):
    """Planes the persistent kernel cannot hold (W > 2048 columns; 325 strips of
    4 rows > the co-resident CTAs) run the one-launch-per-plane fallback."""
    rng = np.random.default_rng(29)
    img = dyadic_image(rng, shape)
    mask = point_mask(shape)
    for lam in (0.0, 1.0):
        g = gd.generalized_geodesic(img, mask, (1.0, 1.0, 1.0), lam, 1e10, 1)
        r = oracle.generalized_geodesic(img, mask, (1.0, 1.0, 1.0), lam, 1e10, 1)
        assert bitwise_equal(g, r), parity(g, r)


@pytest.mark.parametrize("lam", [0.0, 1.0])
def test_gsf(gd, oracle, lam):
    shape = (24, 32, 28)
    img = dyadic_image(np.random.default_rng(17), shape)
    zz, yy, xx = np.meshgrid(*[np.arange(s) for s in shape], indexing="ij")
    ball = (((zz - 12) ** 2 + (yy - 16) ** 2 + (xx - 14) ** 2) <= 64).astype(np.float32)
    ball[12, 16, 14] = 0.0  # a hole the closing must fill
    g, gr, gce = gd.gsf(img, ball, None, lam, 1e10, 2, 2.0)
    r, rr, rce = oracle.gsf(img, ball, None, lam, 1e10, 2, 2.0)
    assert bitwise_equal(g, r)
    assert (gr, gce) == (rr, rce)


def test_gsf_complement_empty(gd, oracle):
    # transforms.cpp:213-219 / test_transforms.cpp:380-391
    img = np.zeros((1, 5), np.float32)
    mask = np.array([[1, 1, 0, 1, 1]], np.float32)
    g, rounds, ce = gd.gsf(img, mask, None, 0.0, 1e10, 2, 1.0)
    assert np.all(g == 1.0) and ce and rounds == 2


def test_scan_to_fixpoint(gd, oracle):
    rng = np.random.default_rng(19)
    shape = (15, 15)
    img = dyadic_image(rng, shape)
    d0 = seed_init(rng, shape, 1)
    g, gr, gc, gl = gd.scan_to_fixpoint(img, d0, None, 1.0, 100, 1e-6)
    r, rr, rc, rl = oracle.scan_to_fixpoint(img, d0, None, 1.0, max_rounds=100, tol=1e-6)
    assert bitwise_equal(g, r) and (gr, gc) == (rr, rc) and gl == rl


# ---- known answers restated from the reference's own tests -----------------
def test_known_top_bottom_3x3(gd):
    # test_scan_parallel.cpp:99-114
    img = np.zeros((3, 3), np.float32)
    init = np.full((3, 3), 1e10, np.float32)
    init[1, 1] = 0
    d = gd.directional_pass(init, img, 1, 1, None, 0.0)
    assert np.array_equal(d[:2], init[:2])
    r2 = np.float32(math.sqrt(2.0))
    assert np.allclose(d[2], [r2, 1.0, r2], rtol=1e-6)


def test_known_one_ring_chamfer(gd):
    # test_scan_parallel.cpp:159-170
    img = np.zeros((3, 3), np.float32)
    init = np.full((3, 3), 1e10, np.float32)
    init[1, 1] = 0
    d = gd.parallel_scan(img, init, None, 0.0, 1)
    r2 = math.sqrt(2.0)
    assert np.allclose(d.reshape(-1), [r2, 1, r2, 1, 0, 1, r2, 1, r2], rtol=1e-6)


def test_iterations_compose_bitwise(gd):
    # test_scan_parallel.cpp:172-184
    rng = np.random.default_rng(67)
    img = dyadic_image(rng, (8, 8))
    init = seed_init(rng, (8, 8), 2)
    two = gd.parallel_scan(img, init, None, 0.5, 2)
    one = gd.parallel_scan(img, gd.parallel_scan(img, init, None, 0.5, 1), None, 0.5, 1)
    assert bitwise_equal(two, one)


def test_all_zero_is_fixed(gd):
    # test_scan_parallel.cpp:116-126
    img = np.full((4, 4), 0.5, np.float32)
    zeros = np.zeros((4, 4), np.float32)
    for axis, o in ((1, 1), (1, -1), (2, 1), (2, -1)):
        assert bitwise_equal(gd.directional_pass(zeros, img, axis, o, None, 1.0), zeros)


def test_invalid_arguments(gd):
    img = np.zeros((2, 2), np.float32)
    with pytest.raises(gd.InvalidArgument):
        gd.directional_pass(img, img, 0, 1)  # 3D direction on a 2D grid
    with pytest.raises(gd.InvalidArgument):
        gd.generalized_geodesic(img, np.full((2, 2), 2.0, np.float32))  # mask out of range
    with pytest.raises(gd.InvalidArgument):
        gd.parallel_scan(img, img, None, 1.5, 1)
    with pytest.raises(gd.InvalidArgument):
        gd.gsf(img, img, None, 1.0, 1e10, 2, -0.5)


# ---- committed golden vectors from the unmodified reference -----------------
import glob  # noqa: E402
import os  # noqa: E402

_GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


@pytest.mark.parametrize("path", _GOLDEN, ids=[os.path.basename(p) for p in _GOLDEN])
def test_cuda_matches_golden(gd, path):
    from tests.test_oracle import run_fixture
    f = np.load(path)
    lam = float(f["lam"])
    got = run_fixture(gd, f)
    if lam in (0.0, 1.0) or str(f["kind"]) == "gsf":
        assert bitwise_equal(got, f["out"]), parity(got, f["out"])
    else:
        ok, *_ = parity(got, f["out"])
        assert ok
        gd.set_exact_blend(True)
        try:
            assert bitwise_equal(run_fixture(gd, f), f["out"])
        finally:
            gd.set_exact_blend(False)


@pytest.mark.parametrize("lam", LAMBDAS)
def test_layout_planner_batch(gd, oracle, lam):
    """A batch of narrow volumes: the planner runs the z pass on [x][z][y] (rows
    along the short x axis: 6 strips per volume instead of 12, one launch group
    instead of two), rotating the distance between layouts; every volume stays
    bit-exact / within tolerance."""
    rng = np.random.default_rng(43)
    B, shape = 64, (40, 48, 24)
    imgs = dyadic_image(rng, (B,) + shape)
    masks = np.ones((B,) + shape, np.float32)
    for b in range(B):
        masks[b].reshape(-1)[rng.integers(0, masks[b].size)] = 0.0
    sp = (1.0, 1.3, 2.5)
    gd.launch_log(reset=True)
    g = gd.generalized_geodesic_batched(imgs, masks, sp, lam, 1e10, 2)
    log = [r for r in gd.launch_log(reset=True) if r["f64"] == 0]
    assert {r["layout"] for r in log if r["axis"] == 0} == {1}, log
    for b in range(0, B, 9):
        _check(g[b], oracle.generalized_geodesic(imgs[b], masks[b], sp, lam, 1e10, 2), lam)


def test_layout_rotations_single_passes(gd, oracle):
    """Every single directional pass, including x passes that the planner may
    put on either rotated layout, against the oracle on a non-cube ragged grid."""
    rng = np.random.default_rng(47)
    shape, sp = (13, 22, 9), (1.0, 0.7, 1.9)
    img = dyadic_image(rng, shape)
    d0 = seed_init(rng, shape, 3)
    for axis in range(3):
        for o in (1, -1):
            for lam in LAMBDAS:
                _check(gd.directional_pass(d0, img, axis, o, sp, lam),
                       oracle.directional_pass(d0, img, axis, o, sp, lam), lam)
