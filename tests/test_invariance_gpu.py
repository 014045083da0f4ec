"""Launch-configuration invariance — the reference's worker-count invariance
(test_scan_parallel.cpp:186-205, acceptance A3) re-expressed for the GPU: the
output must be bitwise identical whatever the cluster size (L2-only links,
DSMEM clusters of 2 / 4), the strip shape (one or two rows per warp), the
storage-layout plan (planner or fixed), or the plane-step fallback -- for every
lambda, including blend, whose f32 result is not the reference's bit pattern but
must not depend on how the work was split.  Each setting runs in its own
process (the switches are read once per process)."""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import os, sys
sys.path.insert(0, os.environ["GD_ROOT"])
import numpy as np
import paper_2208_00001_b200 as gd
from tests.helpers import dyadic_image, point_mask
outs = []
for shape, sp in (((10, 288, 300), (1.0, 1.0, 2.5)), ((24, 17, 70), (1.3, 1.0, 0.7))):
    img = dyadic_image(np.random.default_rng(5), shape)
    m = point_mask(shape)
    for lam in (0.0, 0.7, 1.0):
        outs.append(gd.generalized_geodesic(img, m, sp, lam, 1e10, 2))
    imgs = dyadic_image(np.random.default_rng(6), (6,) + shape)
    masks = np.stack([point_mask(shape)] * 6)
    outs.append(gd.generalized_geodesic_batched(imgs, masks, sp, 1.0, 1e10, 1))
np.savez(os.environ["GD_OUT"], *outs)
"""

SETTINGS = {
    "default": {},
    "l2_links_only": {"GEODIST_SWEEP_CLUSTER": "0"},
    "clusters_of_2": {"GEODIST_SWEEP_CLUSTER": "2"},
    "clusters_of_4": {"GEODIST_SWEEP_CLUSTER": "4"},
    "one_row_per_warp": {"GEODIST_SWEEP_RW": "1"},
    "two_rows_per_warp": {"GEODIST_SWEEP_RW": "2"},
    "fixed_layouts": {"GEODIST_LAYOUT_PLAN": "0"},
    "plane_step": {"GEODIST_SWEEP_FALLBACK": "1"},
}


def test_outputs_identical_across_launch_configurations():
    results = {}
    with tempfile.TemporaryDirectory() as td:
        for name, env in SETTINGS.items():
            out = os.path.join(td, name + ".npz")
            e = dict(os.environ, GD_ROOT=ROOT, GD_OUT=out, **env)
            r = subprocess.run([sys.executable, "-c", CHILD], env=e, capture_output=True,
                               text=True, timeout=900)
            assert r.returncode == 0, (name, r.stdout[-2000:], r.stderr[-2000:])
            f = np.load(out)
            results[name] = [f[k] for k in sorted(f.files, key=lambda s: int(s.split("_")[1]))]
    base = results["default"]
    for name, arrs in results.items():
        assert len(arrs) == len(base)
        for i, (a, b) in enumerate(zip(arrs, base)):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (name, i)
