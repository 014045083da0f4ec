"""Every transform of transforms.hpp on the GPU against the unmodified reference.

geodesic_distance, euclidean_distance, signed_geodesic, geodesic_dilate,
geodesic_erode, gsf and generalized_geodesic (transforms.cpp:74-238), each in
the reference's two ScanPolicy modes -- a fixed number of iterations and
to_fixpoint (rounds until the largest change <= tol) -- with hard seeds,
thresholds, counts and the signed subtraction as device kernels.  Bit-exact for
lambda in {0, 1} (and blend in exact mode); the TransformStats (rounds,
converged, complement_empty) must match too.  Edge cases from
test_transforms.cpp: empty seeds, an empty mask or complement for the signed
transform, theta = 0, an erode whose complement is empty.
"""
import numpy as np
import pytest

from tests.helpers import bitwise_equal, dyadic_image, parity

pytestmark = pytest.mark.gpu

TRANSFORMS = ["generalized_geodesic", "geodesic_distance", "euclidean_distance",
              "signed_geodesic", "geodesic_dilate", "geodesic_erode", "gsf"]
SHAPES = [((11, 13), (1.0, 1.5)), ((9, 10, 13), (1.0, 1.0, 2.5)), ((6, 37, 41), (1.3, 1.0, 0.7))]


def _inputs(shape, which, seed):
    rng = np.random.default_rng(seed)
    img = dyadic_image(rng, shape)
    if which == "generalized_geodesic":
        mask = np.ones(shape, np.float32)
        mask.reshape(-1)[rng.integers(0, mask.size, 2)] = 0.0
        mask.reshape(-1)[rng.integers(0, mask.size, 3)] = 0.5  # soft values
    elif which in ("geodesic_distance", "euclidean_distance"):
        mask = np.zeros(shape, np.float32)
        mask.reshape(-1)[rng.integers(0, mask.size, 2)] = 1.0
    else:  # binary blob masks
        mask = (rng.random(shape) < 0.35).astype(np.float32)
    return img, mask


@pytest.mark.parametrize("which", TRANSFORMS)
@pytest.mark.parametrize("shape,spacing", SHAPES, ids=["2d", "3d", "3d_ragged"])
@pytest.mark.parametrize("lam", [0.0, 0.6, 1.0])
@pytest.mark.parametrize("fixpoint", [False, True], ids=["iters", "fixpoint"])
def test_transform_matches_reference(gd, ref, which, shape, spacing, lam, fixpoint):
    if which == "euclidean_distance" and lam != 0.0:
        pytest.skip("euclidean_distance has no lambda")
    img, mask = _inputs(shape, which, hash((which, shape, lam)) % 2**32)
    kw = dict(spacing=spacing, lam=lam, nu=1e10, iterations=2, theta=1.5,
              to_fixpoint=fixpoint, max_rounds=50, tol=1e-6)
    exact = fixpoint and 0.0 < lam < 1.0  # fixpoint round counts need identical arithmetic
    gd.set_exact_blend(exact)
    try:
        got, gst = gd.transform(which, img, mask, **kw)
    finally:
        gd.set_exact_blend(False)
    want, rst = ref.transform(which, img, mask, **kw)
    if lam in (0.0, 1.0) or exact or which in ("geodesic_dilate", "geodesic_erode", "gsf"):
        assert bitwise_equal(got, want), parity(got, want)
    else:
        ok, *_ = parity(got, want)
        assert ok, parity(got, want)
    if lam in (0.0, 1.0) or exact:
        assert gst == rst, (gst, rst)


@pytest.mark.parametrize("which", ["geodesic_distance", "euclidean_distance"])
def test_empty_seeds(gd, which):
    z = np.zeros((4, 5), np.float32)
    with pytest.raises(gd.EmptySeedsError):
        gd.transform(which, z, z)


def test_signed_geodesic_empty_sides(gd, ref):
    img = np.zeros((4, 5), np.float32)
    for mask in (np.zeros((4, 5), np.float32), np.ones((4, 5), np.float32)):
        with pytest.raises(gd.EmptySeedsError):
            gd.signed_geodesic(img, mask)
        with pytest.raises(Exception):
            ref.transform("signed_geodesic", img, mask)


def test_signed_geodesic_axial_example(gd):
    # test_transforms.cpp:206-248: 1 x 5 row, mask on the first two cells, lambda = 0
    img = np.zeros((1, 5), np.float32)
    mask = np.array([[1, 1, 0, 0, 0]], np.float32)
    s = gd.signed_geodesic(img, mask, None, 0.0, 2)
    assert np.allclose(s[0], [-2, -1, 1, 2, 3])
    flipped = gd.signed_geodesic(img, 1.0 - mask, None, 0.0, 2)
    assert np.array_equal(flipped, -s)  # exact antisymmetry (A7)


def test_erode_complement_empty_and_theta0(gd, ref):
    img = dyadic_image(np.random.default_rng(3), (6, 7))
    ones = np.ones((6, 7), np.float32)
    got, st = gd.transform("geodesic_erode", img, ones, theta=1.0)
    want, rst = ref.transform("geodesic_erode", img, ones, theta=1.0)
    assert bitwise_equal(got, want) and st == rst and st["complement_empty"]
    m = (np.random.default_rng(4).random((6, 7)) < 0.5).astype(np.float32)
    got, _ = gd.transform("gsf", img, m, theta=0.0)  # theta = 0: identity on binary masks
    assert bitwise_equal(got, m)


def test_transforms_on_the_device_async(gd, ref):
    """The device-memory entries of the new transforms enqueue without blocking
    and report empty seeds as a deferred error."""
    import ctypes as C

    import torch
    shape = (8, 12, 16)
    img, mask = _inputs(shape, "signed_geodesic", 11)
    d_img, d_mask = torch.from_numpy(img).cuda(), torch.from_numpy(mask).cuda()
    d_out = torch.empty_like(d_img)
    g = gd._grid(shape, None)
    L = gd.lib()
    gd._check(L.gd_signed_geodesic(C.byref(g), C.c_void_p(d_img.data_ptr()),
                                   C.c_void_p(d_mask.data_ptr()), 1.0, 2, None,
                                   C.c_void_p(d_out.data_ptr()), gd.GD_MEM_DEVICE,
                                   gd.device._stream(None), None))
    gd.device.synchronize()
    want, _ = ref.transform("signed_geodesic", img, mask, lam=1.0, iterations=2)
    assert bitwise_equal(d_out.cpu().numpy(), want)
    zeros = torch.zeros(shape, device="cuda")
    gd._check(L.gd_euclidean_distance(C.byref(g), C.c_void_p(zeros.data_ptr()), 2, None,
                                      C.c_void_p(d_out.data_ptr()), gd.GD_MEM_DEVICE,
                                      gd.device._stream(None), None))
    with pytest.raises(gd.EmptySeedsError):
        gd.device.synchronize()


@pytest.mark.parametrize("lam", [0.0, 1.0])
@pytest.mark.parametrize("theta", [0.0, 1.5, 4.0])
def test_gsf_symmetric_is_the_reference_composition(gd, ref, lam, theta):
    """The upstream-style 4-transform filter equals the reference's own calls
    composed: dilate -> erode (its gsf) -> erode -> dilate."""
    shape, sp = (10, 24, 22), (1.0, 1.0, 2.5)
    img, mask = _inputs(shape, "gsf", 21)
    got, st = gd.transform("gsf_symmetric", img, mask, sp, lam, 1e10, 2, theta)
    kw = dict(spacing=sp, lam=lam, nu=1e10, iterations=2, theta=theta)
    d1, r1 = ref.transform("geodesic_dilate", img, mask, **kw)
    e1, r2 = ref.transform("geodesic_erode", img, d1, **kw)
    e2, r3 = ref.transform("geodesic_erode", img, e1, **kw)
    want, r4 = ref.transform("geodesic_dilate", img, e2, **kw)
    assert bitwise_equal(got, want)
    assert st["rounds"] == r1["rounds"] + r2["rounds"] + r3["rounds"] + r4["rounds"]
