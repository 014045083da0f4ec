"""CPU: the geodist_b200 CLI (bin/geodist_b200, csrc/cli.cpp) and its FGD1 I/O
(csrc/io.cpp) on the paths that need no GPU: `compare` on FGD1 files written
here in the reference's layout (io.hpp:43-49), exit codes (0 / 1 over tolerance
/ 2 usage / 3 I/O, tools/main.cpp:28-31), malformed-file diagnostics, and a
compute call failing loudly without a device (no CPU fallback)."""
import os
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2208_00001_b200", "bin", "geodist_b200")


def fgd1(path, a, spacing=None):
    a = np.ascontiguousarray(a, np.float32)
    sp = spacing or (1.0,) * a.ndim
    with open(path, "wb") as f:
        f.write(b"FGD1" + struct.pack("<I", a.ndim) + struct.pack(f"<{a.ndim}I", *a.shape) +
                struct.pack(f"<{a.ndim}f", *sp) + a.astype("<f4").tobytes())


def run(*args):
    if not os.path.exists(CLI):
        pytest.fail(f"{CLI} not built (make -C paper_2208_00001_b200)")
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=60)


def test_compare_identical_and_differing(tmp_path):
    a = np.arange(12, dtype=np.float32).reshape(3, 4)
    b = a.copy()
    b[1, 2] += 0.5
    fgd1(tmp_path / "a.fgd", a)
    fgd1(tmp_path / "b.fgd", b)
    same = run("compare", "--a", str(tmp_path / "a.fgd"), "--b", str(tmp_path / "a.fgd"))
    assert same.returncode == 0 and "max_abs_diff=0 " in same.stdout
    diff = run("compare", "--a", str(tmp_path / "a.fgd"), "--b", str(tmp_path / "b.fgd"),
               "--tol", "1e-3")
    assert diff.returncode == 1
    assert "at=(1,2)" in diff.stdout and "cells_over_tol=1" in diff.stdout


def test_io_errors_and_usage(tmp_path):
    (tmp_path / "bad.fgd").write_bytes(b"NOPE" + b"\0" * 20)
    fgd1(tmp_path / "a.fgd", np.zeros((2, 2), np.float32))
    r = run("compare", "--a", str(tmp_path / "bad.fgd"), "--b", str(tmp_path / "a.fgd"))
    assert r.returncode == 3 and "bad magic" in r.stderr
    r = run("compare", "--a", str(tmp_path / "missing.fgd"), "--b", str(tmp_path / "a.fgd"))
    assert r.returncode == 3
    assert run("compare", "--a", str(tmp_path / "a.fgd")).returncode == 2  # --b missing
    assert run("frobnicate").returncode == 2
    r = run("compute", "--input", str(tmp_path / "a.fgd"), "--seeds", str(tmp_path / "a.fgd"),
            "--mode", "gsf", "--output", str(tmp_path / "o.fgd"))
    assert r.returncode == 2 and "--theta is required" in r.stderr


def test_compute_without_gpu_fails_loudly(tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    img = np.zeros((4, 5), np.float32)
    seeds = np.zeros((4, 5), np.float32)
    seeds[2, 2] = 1.0
    fgd1(tmp_path / "i.fgd", img)
    fgd1(tmp_path / "s.fgd", seeds)
    r = run("compute", "--input", str(tmp_path / "i.fgd"), "--seeds", str(tmp_path / "s.fgd"),
            "--mode", "euclidean", "--output", str(tmp_path / "o.fgd"))
    assert r.returncode == 4 and "no CUDA device" in r.stderr
    assert not (tmp_path / "o.fgd").exists()
