"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the two CPU checkers.

* ``RefLib``  — the unmodified reference (``oracle/_ref/libgeodist_ref.so``,
  built by ``oracle/Makefile`` from /root/reference/proj/src).
* ``COracle`` — the plain-C restatement (``oracle/_build/libgd_oracle.so``).

Both expose the same numpy-level calls so tests can swap them.  Only tests/,
``__graft_entry__.smoke()`` and bench.py's CPU legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libgeodist_ref.so")
ORACLE_SO = os.path.join(HERE, "_build", "libgd_oracle.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i = C.c_int
_d = C.c_double
_ip = C.POINTER(C.c_int)
_dp = C.POINTER(C.c_double)


class OracleError(RuntimeError):
    pass


class InvalidArgument(OracleError, ValueError):
    pass


class EmptySeeds(OracleError):
    pass


def build(target: str = "all") -> None:
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


def _arr_i(v):
    return (C.c_int * 3)(*v)


def _arr_d(v):
    return (C.c_double * 3)(*[float(x) for x in v])


def _canon(image: np.ndarray, spacing):
    ndim = image.ndim
    if ndim not in (2, 3):
        raise InvalidArgument("grid rank must be 2 or 3")
    if spacing is None:
        spacing = (1.0,) * ndim
    if len(spacing) != ndim:
        raise InvalidArgument("spacing length does not match rank")
    return ndim, _arr_i(image.shape), _arr_d(spacing)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class _Base:
    def _check(self, rc: int):
        if rc == 0:
            return
        msg = self._msg()
        if rc == 1:
            raise InvalidArgument(msg)
        if rc == 2:
            raise EmptySeeds(msg)
        raise OracleError(msg)

    def _msg(self) -> str:
        return "invalid argument"


class RefLib(_Base):
    """The unmodified reference library behind a C shim (oracle/ref_shim.cpp)."""

    def __init__(self, path: str = REF_SO, workers: int | None = None):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.workers = workers or os.cpu_count() or 1
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_generalized_geodesic.argtypes = [_i, _ip, _dp, _f32p, _f32p, _d, _d, _i, _i, _f32p, _ip]
        L.ref_gsf.argtypes = [_i, _ip, _dp, _f32p, _f32p, _d, _d, _i, _d, _i, _f32p, _ip, _ip]
        L.ref_directional_pass.argtypes = [_i, _ip, _dp, _f32p, _f32p, _i, _i, _d, _i]
        L.ref_parallel_scan.argtypes = [_i, _ip, _dp, _f32p, _f32p, _d, _i, _i]
        L.ref_serial_scan.argtypes = [_i, _ip, _dp, _f32p, _f32p, _d, _i]
        L.ref_scan_to_fixpoint.argtypes = [_i, _ip, _dp, _f32p, _f32p, _d, _i, _i, _d, _i, _ip, _ip, _dp]
        L.ref_geodesic_distance.argtypes = [_i, _ip, _dp, _f32p, _f32p, _d, _i, _i, _f32p]
        L.ref_euclidean_distance.argtypes = [_i, _ip, _dp, _f32p, _i, _i, _f32p]
        L.ref_signed_geodesic.argtypes = [_i, _ip, _dp, _f32p, _f32p, _d, _i, _i, _f32p]
        L.ref_dijkstra_exact.argtypes = [_i, _ip, _dp, _f32p, _f32p, _d, _f32p]
        L.ref_pass_offsets.argtypes = [_i, _dp, _i, _i, _ip, _dp, _ip]
        L.ref_transform_ex.argtypes = [_i, _i, _ip, _dp, _f32p, _f32p, _d, _d, _i, _d, _i, _i, _d,
                                       _i, _f32p, _ip, _ip, _ip]

    def _msg(self):
        return self.lib.ref_last_error().decode()

    def generalized_geodesic(self, image, mask, spacing=None, lam=1.0, nu=1e10, iterations=2,
                             workers=None):
        image, mask = _f32(image), _f32(mask)
        ndim, dims, sp = _canon(image, spacing)
        out = np.empty_like(image)
        rounds = C.c_int(0)
        self._check(self.lib.ref_generalized_geodesic(ndim, dims, sp, image, mask, lam, nu,
                                                      iterations, workers or self.workers, out,
                                                      C.byref(rounds)))
        return out

    def gsf(self, image, mask, spacing=None, lam=1.0, nu=1e10, iterations=2, theta=0.0,
            workers=None):
        image, mask = _f32(image), _f32(mask)
        ndim, dims, sp = _canon(image, spacing)
        out = np.empty_like(image)
        rounds, ce = C.c_int(0), C.c_int(0)
        self._check(self.lib.ref_gsf(ndim, dims, sp, image, mask, lam, nu, iterations, theta,
                                     workers or self.workers, out, C.byref(rounds), C.byref(ce)))
        return out, rounds.value, bool(ce.value)

    def directional_pass(self, dist, image, axis, orientation, spacing=None, lam=1.0,
                         workers=None):
        image = _f32(image)
        d = _f32(dist).copy()
        ndim, dims, sp = _canon(image, spacing)
        self._check(self.lib.ref_directional_pass(ndim, dims, sp, image, d, axis, orientation,
                                                  lam, workers or self.workers))
        return d

    def parallel_scan(self, image, dist, spacing=None, lam=1.0, iterations=2, workers=None):
        image = _f32(image)
        d = _f32(dist).copy()
        ndim, dims, sp = _canon(image, spacing)
        self._check(self.lib.ref_parallel_scan(ndim, dims, sp, image, d, lam, iterations,
                                               workers or self.workers))
        return d

    def scan_to_fixpoint(self, image, dist, spacing=None, lam=1.0, engine=1, max_rounds=100,
                         tol=1e-6, workers=None):
        image = _f32(image)
        d = _f32(dist).copy()
        ndim, dims, sp = _canon(image, spacing)
        ru, cv, lc = C.c_int(0), C.c_int(0), C.c_double(0)
        self._check(self.lib.ref_scan_to_fixpoint(ndim, dims, sp, image, d, lam, engine,
                                                  max_rounds, tol, workers or self.workers,
                                                  C.byref(ru), C.byref(cv), C.byref(lc)))
        return d, ru.value, bool(cv.value), lc.value

    TRANSFORMS = ("generalized_geodesic", "geodesic_distance", "euclidean_distance",
                  "signed_geodesic", "geodesic_dilate", "geodesic_erode", "gsf")

    def transform(self, which, image, mask, spacing=None, lam=1.0, nu=1e10, iterations=2,
                  theta=0.0, to_fixpoint=False, max_rounds=100, tol=1e-6, workers=None):
        """Any transforms.hpp transform with a full ScanPolicy; returns
        (out, {rounds, converged, complement_empty})."""
        image, mask = _f32(image), _f32(mask)
        ndim, dims, sp = _canon(mask, spacing)
        out = np.empty_like(mask)
        ru, cv, ce = C.c_int(0), C.c_int(0), C.c_int(0)
        self._check(self.lib.ref_transform_ex(self.TRANSFORMS.index(which), ndim, dims, sp, image,
                                              mask, lam, nu, iterations, theta,
                                              1 if to_fixpoint else 0, max_rounds, tol,
                                              workers or self.workers, out, C.byref(ru),
                                              C.byref(cv), C.byref(ce)))
        return out, {"rounds": ru.value, "converged": bool(cv.value),
                     "complement_empty": bool(ce.value)}

    def dijkstra_exact(self, image, init, spacing=None, lam=1.0):
        image, init = _f32(image), _f32(init)
        ndim, dims, sp = _canon(image, spacing)
        out = np.empty_like(image)
        self._check(self.lib.ref_dijkstra_exact(ndim, dims, sp, image, init, lam, out))
        return out

    def pass_offsets(self, ndim, spacing, axis, orientation):
        dzyx = (C.c_int * 27)()
        rho = (C.c_double * 9)()
        n = C.c_int(0)
        self._check(self.lib.ref_pass_offsets(ndim, _arr_d(spacing), axis, orientation, dzyx,
                                              rho, C.byref(n)))
        return [(dzyx[3 * k], dzyx[3 * k + 1], dzyx[3 * k + 2], rho[k]) for k in range(n.value)]


class COracle(_Base):
    """The plain-C restatement (oracle/gd_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build("oracle")
        self.lib = C.CDLL(path)
        L = self.lib
        L.gdo_pass_offsets.argtypes = [_i, _dp, _i, _i, _ip, _dp, _ip]
        L.gdo_directional_pass.argtypes = [_i, _ip, _dp, _f32p, _f32p, _i, _i, _d]
        L.gdo_parallel_scan.argtypes = [_i, _ip, _dp, _f32p, _f32p, _d, _i]
        L.gdo_generalized_geodesic.argtypes = [_i, _ip, _dp, _f32p, _f32p, _d, _d, _i, _f32p]
        L.gdo_gsf.argtypes = [_i, _ip, _dp, _f32p, _f32p, _d, _d, _i, _d, _f32p, _ip, _ip]
        L.gdo_scan_to_fixpoint.argtypes = [_i, _ip, _dp, _f32p, _f32p, _d, _i, _d, _ip, _ip, _dp]

    def generalized_geodesic(self, image, mask, spacing=None, lam=1.0, nu=1e10, iterations=2,
                             workers=None):
        image, mask = _f32(image), _f32(mask)
        ndim, dims, sp = _canon(image, spacing)
        out = np.empty_like(image)
        self._check(self.lib.gdo_generalized_geodesic(ndim, dims, sp, image, mask, lam, nu,
                                                      iterations, out))
        return out

    def gsf(self, image, mask, spacing=None, lam=1.0, nu=1e10, iterations=2, theta=0.0,
            workers=None):
        image, mask = _f32(image), _f32(mask)
        ndim, dims, sp = _canon(image, spacing)
        out = np.empty_like(image)
        rounds, ce = C.c_int(0), C.c_int(0)
        self._check(self.lib.gdo_gsf(ndim, dims, sp, image, mask, lam, nu, iterations, theta,
                                     out, C.byref(rounds), C.byref(ce)))
        return out, rounds.value, bool(ce.value)

    def directional_pass(self, dist, image, axis, orientation, spacing=None, lam=1.0,
                         workers=None):
        image = _f32(image)
        d = _f32(dist).copy()
        ndim, dims, sp = _canon(image, spacing)
        self._check(self.lib.gdo_directional_pass(ndim, dims, sp, image, d, axis, orientation,
                                                  lam))
        return d

    def parallel_scan(self, image, dist, spacing=None, lam=1.0, iterations=2, workers=None):
        image = _f32(image)
        d = _f32(dist).copy()
        ndim, dims, sp = _canon(image, spacing)
        self._check(self.lib.gdo_parallel_scan(ndim, dims, sp, image, d, lam, iterations))
        return d

    def scan_to_fixpoint(self, image, dist, spacing=None, lam=1.0, engine=1, max_rounds=100,
                         tol=1e-6, workers=None):
        image = _f32(image)
        d = _f32(dist).copy()
        ndim, dims, sp = _canon(image, spacing)
        ru, cv, lc = C.c_int(0), C.c_int(0), C.c_double(0)
        self._check(self.lib.gdo_scan_to_fixpoint(ndim, dims, sp, image, d, lam, max_rounds, tol,
                                                  C.byref(ru), C.byref(cv), C.byref(lc)))
        return d, ru.value, bool(cv.value), lc.value

    def pass_offsets(self, ndim, spacing, axis, orientation):
        dzyx = (C.c_int * 27)()
        rho = (C.c_double * 9)()
        n = C.c_int(0)
        self._check(self.lib.gdo_pass_offsets(ndim, (C.c_double * 3)(*spacing), axis,
                                              orientation, dzyx, rho, C.byref(n)))
        return [(dzyx[3 * k], dzyx[3 * k + 1], dzyx[3 * k + 2], rho[k]) for k in range(n.value)]


# ---------------------------------------------------------------------------
# Synthetic inputs; shared by tests and bench.py.
# ---------------------------------------------------------------------------
def splitmix64_unit(n: int, seed: int) -> np.ndarray:
    """tools/main.cpp:67-81: f32((next() >> 40) * 2^-24), row-major fill."""
    with np.errstate(over="ignore"):
        gamma = np.uint64(0x9E3779B97F4A7C15)
        idx = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(seed) + idx * gamma
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return ((z >> np.uint64(40)).astype(np.float64) * 2.0 ** -24).astype(np.float32)


def bench_seed(ndim: int, size: int) -> int:
    """tools/main.cpp:312-314."""
    return 0x67656F64697374 ^ (ndim << 32) ^ size
