"""CPU: the C-ABI library loads, exports every symbol include/geodist_b200.h
declares (and the C++ drop-in API), validates arguments on the host before
touching the device, and fails loudly (no CPU fallback) without a GPU."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "geodist_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(gd_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_symbols()
    for must in ("gd_generalized_geodesic", "gd_generalized_geodesic_batched", "gd_gsf",
                 "gd_directional_pass", "gd_parallel_scan", "gd_scan_to_fixpoint",
                 "gd_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(gd):
    lib = gd.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_cpp_dropin_symbols_exported(gd):
    out = subprocess.run(["nm", "-D", "-C", "--defined-only", gd.LIB_PATH], capture_output=True,
                         text=True).stdout
    for sym in ("geodist::generalized_geodesic(", "geodist::gsf(", "geodist::directional_pass(",
                "geodist::parallel_scan(", "geodist::detail::parallel_scan_inplace(",
                "geodist::detail::directional_pass_inplace(", "geodist::scan_to_fixpoint(",
                "geodist::ScalarGrid::ScalarGrid(", "geodist::pass_neighbor_offsets(",
                "geodist::run_scan(", "geodist::GSF3d(", "geodist::generalised_geodesic3d("):
        assert sym in out, sym


def test_cpp_headers_compile_standalone():
    # a reference caller compiles unchanged against include/geodist/*.hpp
    src = r"""
    #include "geodist/transforms.hpp"
    int use() {
        const int dims[3] = {4, 4, 4};
        const double sp[3] = {1.0, 1.0, 2.5};
        geodist::ScalarGrid img(3, dims, sp, 0.0f), m(3, dims, sp, 1.0f);
        geodist::TransformParams p;
        geodist::ScanPolicy pol;
        geodist::TransformStats st;
        auto d = geodist::generalized_geodesic(img, m, p, pol, &st);
        geodist::GsfParams gp;
        auto g = geodist::gsf(img, m, gp, pol, &st);
        return static_cast<int>(d.size() + g.size());
    }
    """
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                        "-x", "c++", "-"], input=src, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_host_validation_before_device(gd):
    # grid validation happens on the host (ScalarGrid rules, grid.cpp:10-39)
    lib = gd.lib()
    g = gd.gd_grid()
    g.ndim = 4
    rc = lib.gd_parallel_scan(C.byref(g), None, None, 1.0, 1, gd.GD_MEM_HOST, None)
    assert rc == gd.GD_INVALID_ARGUMENT
    g = gd._grid((3, 0), None)
    a = np.zeros(1, np.float32)
    rc = lib.gd_parallel_scan(C.byref(g), gd._ptr(a), gd._ptr(a), 1.0, 1, gd.GD_MEM_HOST, None)
    assert rc == gd.GD_INVALID_ARGUMENT
    assert "extent" in lib.gd_last_error().decode()


def test_no_cpu_fallback(gd):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except Exception:
        pass
    with pytest.raises(gd.CudaError):
        gd.generalized_geodesic(np.zeros((4, 4), np.float32), np.ones((4, 4), np.float32))


def test_python_mirror_validates_shapes(gd):
    with pytest.raises(gd.InvalidArgument):
        gd.generalized_geodesic(np.zeros((4, 4), np.float32), np.ones((4, 5), np.float32))
    with pytest.raises(gd.InvalidArgument):
        gd.directional_pass(np.zeros((4, 4), np.float32), np.zeros((4, 5), np.float32), 1, 1)
