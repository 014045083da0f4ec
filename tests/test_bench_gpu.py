"""bench.py's driver contract on one GPU: one JSON line with the base keys, the
roofline / e2e / gpu_launches / clocks objects, and the reference arm's line on
the same metric and config (short runs; the numbers themselves are judged from
the full runs in profiles/)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-2000:])
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run("--steps", "3", "--warmup", "3", "--no-cpu", "--e2e-steps", "2")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert "512x512x512" in d["config"]["workload"]
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s"
    assert 0.0 < rf["frac"] < 1.0
    assert abs(rf["achieved"] / rf["peak"] - rf["frac"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 2 * 512 ** 3 * 4
    assert e["d2h_bytes_per_step"] == 512 ** 3 * 4
    assert d["gpu_launches"] > 3 * 12  # >= 12 sweeps per transform, 3 timed steps


def test_reference_arm_same_config():
    ours = _run("--steps", "3", "--warmup", "3", "--no-cpu", "--e2e-steps", "2")
    ref = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert ref["impl"] == "reference"
    for k in ("metric", "unit", "higher_is_better"):
        assert ref[k] == ours[k], k
    assert ref["config"]["workload"] == ours["config"]["workload"]
    assert ref["value"] > 0
    assert ref["e2e"]["h2d_bytes_per_step"] == 0 and ref["cpu_baseline"]["cores"] >= 1
