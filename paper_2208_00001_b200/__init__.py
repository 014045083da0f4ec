"""geodist_b200 — B200-native generalised geodesic distance transform.

Python host mirror of the reference's operator interface
(/root/reference/proj/include/geodist/{transforms,scan_parallel}.hpp) over the
C-ABI in ``include/geodist_b200.h``.  Every call runs the sm_100a kernels in
``lib/libgeodist_b200.so``; there is no CPU fallback — importing without the
built library, or calling without a CUDA device, raises.

Host (numpy) calls mirror ``geodist::*`` one-to-one (same argument meaning and
error types: ``InvalidArgument`` for the reference's std::invalid_argument,
``EmptySeedsError`` for geodist::EmptySeedsError).  ``device`` holds the same
calls on CUDA tensors (torch) enqueued on the current stream.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

__all__ = [
    "GeodistError", "InvalidArgument", "EmptySeedsError", "UnsupportedShape", "CudaError",
    "generalized_geodesic", "generalized_geodesic_batched", "gsf", "directional_pass",
    "parallel_scan", "scan_to_fixpoint", "generalised_geodesic2d", "generalised_geodesic3d",
    "GSF2d", "GSF3d", "set_exact_blend", "kernel_launches", "device", "LIB_PATH", "transform",
    "geodesic_distance", "euclidean_distance", "signed_geodesic", "geodesic_dilate",
    "geodesic_erode", "gsf_symmetric",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GEODIST_LIB") or os.path.join(HERE, "lib", "libgeodist_b200.so")

GD_OK, GD_INVALID_ARGUMENT, GD_EMPTY_SEEDS, GD_CUDA_ERROR, GD_UNSUPPORTED = range(5)
GD_MEM_HOST, GD_MEM_DEVICE = 0, 1


class GeodistError(RuntimeError):
    pass


class InvalidArgument(GeodistError, ValueError):
    pass


class EmptySeedsError(GeodistError):
    pass


class CudaError(GeodistError):
    pass


class UnsupportedShape(GeodistError):
    pass


class gd_grid(C.Structure):
    _fields_ = [("ndim", C.c_int), ("dims", C.c_int * 3), ("spacing", C.c_double * 3)]


class gd_launch_rec(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("axis", "npass", "kind", "f64", "path", "rows", "nwv",
                                       "nwu", "cs", "ntu", "nvol", "grid", "tb", "layout")]


class gd_policy(C.Structure):
    _fields_ = [("to_fixpoint", C.c_int), ("max_rounds", C.c_int), ("tol", C.c_double)]


class gd_stats(C.Structure):
    _fields_ = [("rounds", C.c_int), ("converged", C.c_int), ("complement_empty", C.c_int),
                ("last_change", C.c_double), ("kernel_launches", C.c_longlong)]


_lib = None


def lib():
    """The loaded C-ABI library (loaded once; raises if it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (make -C "
                              f"paper_2208_00001_b200); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        vp, d, i, fp = C.c_void_p, C.c_double, C.c_int, C.c_void_p
        gp, sp = C.POINTER(gd_grid), C.POINTER(gd_stats)
        L.gd_generalized_geodesic.argtypes = [gp, fp, fp, d, d, i, fp, i, vp, sp]
        L.gd_generalized_geodesic_batched.argtypes = [gp, i, fp, fp, d, d, i, fp, i, vp, sp]
        L.gd_gsf.argtypes = [gp, fp, fp, d, d, i, d, fp, i, vp, sp]
        L.gd_directional_pass.argtypes = [gp, fp, fp, i, i, d, i, vp]
        L.gd_parallel_scan.argtypes = [gp, fp, fp, d, i, i, vp]
        L.gd_scan_to_fixpoint.argtypes = [gp, fp, fp, d, i, d, i, vp, sp]
        L.gd_set_exact_blend.argtypes = [i]
        L.gd_set_layout_plan.argtypes = [i]
        L.gd_last_error.restype = C.c_char_p
        L.gd_kernel_launches.restype = C.c_longlong
        L.gd_fill_splitmix.argtypes = [fp, C.c_longlong, C.c_ulonglong, vp]
        L.gd_set_device.argtypes = [i]
        L.gd_synchronize.argtypes = [vp]
        pp = C.POINTER(gd_policy)
        L.gd_generalized_geodesic_ex.argtypes = [gp, i, fp, fp, d, d, i, pp, fp, i, vp, sp]
        L.gd_geodesic_distance.argtypes = [gp, fp, fp, d, i, pp, fp, i, vp, sp]
        L.gd_euclidean_distance.argtypes = [gp, fp, i, pp, fp, i, vp, sp]
        L.gd_signed_geodesic.argtypes = [gp, fp, fp, d, i, pp, fp, i, vp, sp]
        L.gd_geodesic_dilate.argtypes = [gp, fp, fp, d, d, d, i, pp, fp, i, vp, sp]
        L.gd_geodesic_erode.argtypes = [gp, fp, fp, d, d, d, i, pp, fp, i, vp, sp]
        L.gd_gsf_ex.argtypes = [gp, fp, fp, d, d, i, d, pp, fp, i, vp, sp]
        L.gd_gsf_symmetric.argtypes = [gp, fp, fp, d, d, i, d, pp, fp, i, vp, sp]
        L.gd_profile_enable.argtypes = [i]
        L.gd_debug_launch_log.argtypes = [C.POINTER(gd_launch_rec), i, i]
        L.gd_profile_read.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_longlong),
                                      C.POINTER(C.c_double), i]
        _lib = L
    return _lib


def _check(rc: int):
    if rc == GD_OK:
        return
    msg = lib().gd_last_error().decode()
    if rc == GD_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if rc == GD_EMPTY_SEEDS:
        raise EmptySeedsError(msg)
    if rc == GD_UNSUPPORTED:
        raise UnsupportedShape(msg)
    raise CudaError(msg)


def _grid(shape, spacing) -> gd_grid:
    ndim = len(shape)
    if spacing is None:
        spacing = (1.0,) * ndim
    if len(spacing) != ndim:
        raise InvalidArgument(f"expected {ndim} spacings, got {len(spacing)}")
    g = gd_grid()
    g.ndim = ndim
    for a in range(min(ndim, 3)):
        g.dims[a] = int(shape[a])
        g.spacing[a] = float(spacing[a])
    return g


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def set_exact_blend(on: bool) -> None:
    """0 < lambda < 1: f64 replica of the reference (bit-exact) instead of f32."""
    lib().gd_set_exact_blend(1 if on else 0)


def set_layout_plan(on: bool) -> None:
    """Per-pass storage-layout planner on (default) / the fixed plan."""
    lib().gd_set_layout_plan(1 if on else 0)


def kernel_launches() -> int:
    return int(lib().gd_kernel_launches())


PROFILE_KINDS = ("sweep", "transpose", "init", "other", "sweep_twin")


def profile_enable(on: bool) -> None:
    lib().gd_profile_enable(1 if on else 0)


def profile_read(reset: bool = True) -> dict:
    """{kind: (ms, launches, algorithmic_bytes)} accumulated since the last reset."""
    n = len(PROFILE_KINDS)
    ms = (C.c_double * n)()
    cnt = (C.c_longlong * n)()
    by = (C.c_double * n)()
    lib().gd_profile_read(ms, cnt, by, 1 if reset else 0)
    return {k: (ms[i], cnt[i], by[i]) for i, k in enumerate(PROFILE_KINDS)}


def profile_log(max_entries: int = 4096):
    """[(kind, ms)] per launch for the launches gathered by profile_read(reset=False)."""
    kinds = (C.c_int * max_entries)()
    ms = (C.c_float * max_entries)()
    n = lib().gd_profile_log(kinds, ms, max_entries)
    return [(PROFILE_KINDS[kinds[i]], ms[i]) for i in range(min(n, max_entries))]


def launch_log(reset: bool = True) -> list:
    """Directional-pass launches since the last reset, oldest first: one dict per
    launch group with the kernel variant that ran (path 0 persistent strip kernel,
    1 row chain, 2 plane-step fallback; rows, warp shape, cluster size cs, ...)."""
    n = lib().gd_debug_launch_log(None, 0, 0)
    buf = (gd_launch_rec * max(n, 1))()
    n = lib().gd_debug_launch_log(buf, n, 1 if reset else 0)
    return [{f: getattr(buf[i], f) for f, _ in gd_launch_rec._fields_} for i in range(n)]


# ---------------------------------------------------------------- host API
def generalized_geodesic(image, soft_mask, spacing=None, lam=1.0, nu=1e10, iterations=2,
                         stats: dict | None = None) -> np.ndarray:
    """geodist::generalized_geodesic (transforms.hpp:62-64)."""
    image, soft_mask = _f32(image), _f32(soft_mask)
    if image.shape != soft_mask.shape:
        raise InvalidArgument("generalized_geodesic: shape mismatch")
    g = _grid(image.shape, spacing)
    out = np.empty_like(image)
    st = gd_stats()
    _check(lib().gd_generalized_geodesic(C.byref(g), _ptr(image), _ptr(soft_mask), lam, nu,
                                         iterations, _ptr(out), GD_MEM_HOST, None, C.byref(st)))
    if stats is not None:
        stats.update(rounds=st.rounds, kernel_launches=st.kernel_launches)
    return out


def _policy(to_fixpoint, max_rounds, tol):
    """ScanPolicy{to_fixpoint, max_rounds, tol} (transforms.hpp:24-30) or None."""
    if not to_fixpoint:
        return None
    p = gd_policy()
    p.to_fixpoint, p.max_rounds, p.tol = 1, int(max_rounds), float(tol)
    return C.byref(p)


def _stats_dict(st):
    return {"rounds": st.rounds, "converged": bool(st.converged),
            "complement_empty": bool(st.complement_empty)}


def _pair(image, mask, what):
    image, mask = _f32(image), _f32(mask)
    if image.shape != mask.shape:
        raise InvalidArgument(f"{what}: shape mismatch")
    return image, mask


def transform(which, image, mask, spacing=None, lam=1.0, nu=1e10, iterations=2, theta=0.0,
              to_fixpoint=False, max_rounds=100, tol=1e-6):
    """Any transforms.hpp transform on the GPU with a full ScanPolicy, mirroring
    the reference's geodist::<which>; returns (out, stats dict).  which:
    generalized_geodesic, geodesic_distance, euclidean_distance (image ignored),
    signed_geodesic, geodesic_dilate, geodesic_erode, gsf."""
    image, mask = _pair(image, mask, which)
    g = _grid(mask.shape, spacing)
    out = np.empty_like(mask)
    st = gd_stats()
    pol = _policy(to_fixpoint, max_rounds, tol)
    L = lib()
    a = (C.byref(g),)
    tail = (_ptr(out), GD_MEM_HOST, None, C.byref(st))
    if which == "generalized_geodesic":
        rc = L.gd_generalized_geodesic_ex(*a, 1, _ptr(image), _ptr(mask), lam, nu, iterations,
                                          pol, *tail)
    elif which == "geodesic_distance":
        rc = L.gd_geodesic_distance(*a, _ptr(image), _ptr(mask), lam, iterations, pol, *tail)
    elif which == "euclidean_distance":
        rc = L.gd_euclidean_distance(*a, _ptr(mask), iterations, pol, *tail)
    elif which == "signed_geodesic":
        rc = L.gd_signed_geodesic(*a, _ptr(image), _ptr(mask), lam, iterations, pol, *tail)
    elif which == "geodesic_dilate":
        rc = L.gd_geodesic_dilate(*a, _ptr(image), _ptr(mask), theta, lam, nu, iterations, pol,
                                  *tail)
    elif which == "geodesic_erode":
        rc = L.gd_geodesic_erode(*a, _ptr(image), _ptr(mask), theta, lam, nu, iterations, pol,
                                 *tail)
    elif which == "gsf":
        rc = L.gd_gsf_ex(*a, _ptr(image), _ptr(mask), lam, nu, iterations, theta, pol, *tail)
    elif which == "gsf_symmetric":
        rc = L.gd_gsf_symmetric(*a, _ptr(image), _ptr(mask), lam, nu, iterations, theta, pol,
                                *tail)
    else:
        raise InvalidArgument(f"unknown transform {which!r}")
    _check(rc)
    return out, _stats_dict(st)


def geodesic_distance(image, seed_mask, spacing=None, lam=1.0, iterations=2, **policy):
    """geodist::geodesic_distance (transforms.hpp:41-44): hard seeds where mask >= 0.5."""
    return transform("geodesic_distance", image, seed_mask, spacing, lam, 1e10, iterations,
                     **policy)[0]


def euclidean_distance(seed_mask, spacing=None, iterations=2, **policy):
    """geodist::euclidean_distance (transforms.cpp:134-141)."""
    seed_mask = _f32(seed_mask)
    return transform("euclidean_distance", seed_mask, seed_mask, spacing, 0.0, 1e10, iterations,
                     **policy)[0]


def signed_geodesic(image, mask, spacing=None, lam=1.0, iterations=2, **policy):
    """geodist::signed_geodesic (transforms.cpp:160-183): d(inside) - d(outside)."""
    return transform("signed_geodesic", image, mask, spacing, lam, 1e10, iterations,
                     **policy)[0]


def geodesic_dilate(image, mask, theta, spacing=None, lam=1.0, nu=1e10, iterations=2, **policy):
    """geodist::geodesic_dilate (transforms.cpp:185-202)."""
    return transform("geodesic_dilate", image, mask, spacing, lam, nu, iterations, theta,
                     **policy)[0]


def geodesic_erode(image, mask, theta, spacing=None, lam=1.0, nu=1e10, iterations=2, **policy):
    """geodist::geodesic_erode (transforms.cpp:204-229)."""
    return transform("geodesic_erode", image, mask, spacing, lam, nu, iterations, theta,
                     **policy)[0]


def generalized_geodesic_batched(images, soft_masks, spacing=None, lam=1.0, nu=1e10,
                                 iterations=2) -> np.ndarray:
    """Batch of independent same-shape grids, leading axis = batch."""
    images, soft_masks = _f32(images), _f32(soft_masks)
    if images.shape != soft_masks.shape:
        raise InvalidArgument("shape mismatch")
    g = _grid(images.shape[1:], spacing)
    out = np.empty_like(images)
    _check(lib().gd_generalized_geodesic_batched(C.byref(g), images.shape[0], _ptr(images),
                                                 _ptr(soft_masks), lam, nu, iterations, _ptr(out),
                                                 GD_MEM_HOST, None, None))
    return out


def gsf(image, soft_mask, spacing=None, lam=1.0, nu=1e10, iterations=2, theta=0.0):
    """geodist::gsf (transforms.hpp:85-86).  Returns (mask, rounds, complement_empty)."""
    image, soft_mask = _f32(image), _f32(soft_mask)
    if image.shape != soft_mask.shape:
        raise InvalidArgument("gsf: shape mismatch")
    g = _grid(image.shape, spacing)
    out = np.empty_like(image)
    st = gd_stats()
    _check(lib().gd_gsf(C.byref(g), _ptr(image), _ptr(soft_mask), lam, nu, iterations, theta,
                        _ptr(out), GD_MEM_HOST, None, C.byref(st)))
    return out, st.rounds, bool(st.complement_empty)


def directional_pass(dist, image, axis, orientation, spacing=None, lam=1.0) -> np.ndarray:
    """geodist::directional_pass (scan_parallel.hpp:20-22); returns the new grid."""
    image = _f32(image)
    d = _f32(dist).copy()
    if d.shape != image.shape:
        raise InvalidArgument("directional_pass: image/distance shape or spacing mismatch")
    g = _grid(image.shape, spacing)
    _check(lib().gd_directional_pass(C.byref(g), _ptr(image), _ptr(d), axis, orientation, lam,
                                     GD_MEM_HOST, None))
    return d


def parallel_scan(image, dist, spacing=None, lam=1.0, iterations=2) -> np.ndarray:
    """geodist::parallel_scan (scan_parallel.hpp:27-28)."""
    image = _f32(image)
    d = _f32(dist).copy()
    if d.shape != image.shape:
        raise InvalidArgument("directional_pass: image/distance shape or spacing mismatch")
    g = _grid(image.shape, spacing)
    _check(lib().gd_parallel_scan(C.byref(g), _ptr(image), _ptr(d), lam, iterations,
                                  GD_MEM_HOST, None))
    return d


def scan_to_fixpoint(image, dist, spacing=None, lam=1.0, max_rounds=100, tol=1e-6):
    """geodist::scan_to_fixpoint, Engine::Parallel.  Returns (dist, rounds, converged, change)."""
    image = _f32(image)
    d = _f32(dist).copy()
    if d.shape != image.shape:
        raise InvalidArgument("scan_to_fixpoint: image/distance shape or spacing mismatch")
    g = _grid(image.shape, spacing)
    st = gd_stats()
    _check(lib().gd_scan_to_fixpoint(C.byref(g), _ptr(image), _ptr(d), lam, max_rounds, tol,
                                     GD_MEM_HOST, None, C.byref(st)))
    return d, st.rounds, bool(st.converged), st.last_change


# Upstream FastGeodis spellings named by the north star.
def generalised_geodesic2d(image, softmask, v, lamb, iter):  # noqa: A002
    return generalized_geodesic(image, softmask, None, lamb, v, iter)


def generalised_geodesic3d(image, softmask, spacing, v, lamb, iter):  # noqa: A002
    return generalized_geodesic(image, softmask, spacing, lamb, v, iter)


def gsf_symmetric(image, softmask, theta, spacing=None, lam=1.0, nu=1e10, iterations=2,
                  **policy):
    """Four chained transforms: opening(closing(M)) with the reference's
    geodesic_dilate / geodesic_erode steps (gd_gsf_symmetric)."""
    return transform("gsf_symmetric", image, softmask, spacing, lam, nu, iterations, theta,
                     **policy)[0]


def GSF2d(image, softmask, theta, v, lamb, iter):  # noqa: A002,N802
    return gsf(image, softmask, None, lamb, v, iter, theta)[0]


def GSF3d(image, softmask, theta, spacing, v, lamb, iter):  # noqa: A002,N802
    return gsf(image, softmask, spacing, lamb, v, iter, theta)[0]


# -------------------------------------------------------------- device API
class device:
    """Same calls on CUDA tensors (torch), enqueued on the current torch stream."""

    @staticmethod
    def set_device(index: int) -> None:
        _check(lib().gd_set_device(int(index)))

    @staticmethod
    def synchronize(stream=None) -> None:
        """Waits for the stream and raises any deferred error of the asynchronous
        calls (InvalidArgument for a soft mask outside [0, 1])."""
        _check(lib().gd_synchronize(device._stream(stream)))

    @staticmethod
    def _bind(t) -> None:
        if t.device.index is not None:
            _check(lib().gd_set_device(int(t.device.index)))

    @staticmethod
    def _validate(shape, **tensors):
        """Every tensor: a contiguous float32 CUDA tensor of exactly `shape`, on the
        device of the first one (the library reads and writes numel() floats)."""
        dev = None
        for name, t in tensors.items():
            if not getattr(t, "is_cuda", False):
                raise InvalidArgument(f"{name}: expected a CUDA tensor")
            if str(t.dtype) != "torch.float32":
                raise InvalidArgument(f"{name}: expected float32, got {t.dtype}")
            if not t.is_contiguous():
                raise InvalidArgument(f"{name}: expected a contiguous tensor")
            if tuple(t.shape) != tuple(shape):
                raise InvalidArgument(f"{name}: shape {tuple(t.shape)} != {tuple(shape)}")
            if dev is None:
                dev = t.device
            elif t.device != dev:
                raise InvalidArgument(f"{name}: on {t.device}, expected {dev}")

    @staticmethod
    def _stream(stream):
        if stream is not None:
            return C.c_void_p(stream)
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)

    @staticmethod
    def generalized_geodesic(image, soft_mask, out, spacing=None, lam=1.0, nu=1e10,
                             iterations=2, batch=None, stream=None):
        """image/soft_mask/out: contiguous float32 CUDA tensors of shape [B?, (D,) H, W]."""
        shape = tuple(image.shape)
        device._validate(shape, image=image, soft_mask=soft_mask, out=out)
        device._bind(image)
        if batch:
            g = _grid(shape[1:], spacing)
        else:
            g = _grid(shape, spacing)
        st = gd_stats()
        _check(lib().gd_generalized_geodesic_batched(
            C.byref(g), int(batch or 1), C.c_void_p(image.data_ptr()),
            C.c_void_p(soft_mask.data_ptr()), lam, nu, iterations, C.c_void_p(out.data_ptr()),
            GD_MEM_DEVICE, device._stream(stream), C.byref(st)))
        return st

    @staticmethod
    def gsf(image, soft_mask, out, spacing=None, lam=1.0, nu=1e10, iterations=2, theta=0.0,
            stream=None):
        device._validate(tuple(image.shape), image=image, soft_mask=soft_mask, out=out)
        device._bind(image)
        g = _grid(tuple(image.shape), spacing)
        st = gd_stats()
        _check(lib().gd_gsf(C.byref(g), C.c_void_p(image.data_ptr()),
                            C.c_void_p(soft_mask.data_ptr()), lam, nu, iterations, theta,
                            C.c_void_p(out.data_ptr()), GD_MEM_DEVICE, device._stream(stream),
                            C.byref(st)))
        return st

    @staticmethod
    def parallel_scan(image, dist, spacing=None, lam=1.0, iterations=2, stream=None):
        device._validate(tuple(image.shape), image=image, dist=dist)
        device._bind(image)
        g = _grid(tuple(image.shape), spacing)
        _check(lib().gd_parallel_scan(C.byref(g), C.c_void_p(image.data_ptr()),
                                      C.c_void_p(dist.data_ptr()), lam, iterations,
                                      GD_MEM_DEVICE, device._stream(stream)))

    @staticmethod
    def fill_splitmix(out, seed: int, stream=None):
        device._validate(tuple(out.shape), out=out)
        device._bind(out)
        _check(lib().gd_fill_splitmix(C.c_void_p(out.data_ptr()), out.numel(),
                                      C.c_ulonglong(seed), device._stream(stream)))
