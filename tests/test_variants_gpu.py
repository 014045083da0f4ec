"""Kernel variants reachable only through tuning switches (read once per process),
checked in a subprocess against the C oracle, each asserting through the launch
log (gd_debug_launch_log) that the variant it asks for really ran: temporal
blocking over plane pairs (GEODIST_SWEEP_TB=1), the one-row-per-warp strip shape
for every cost kind (GEODIST_SWEEP_RW=1), the two-rows-per-warp shape for blend
(RW=2), the plane-step fallback for every plane (GEODIST_SWEEP_FALLBACK=1), DSMEM
halo links inside thread-block clusters of 2, 4 and 8 (GEODIST_SWEEP_CLUSTER=<cs>;
tests/_variant_check.py holds shapes whose strip counts divide by 8), and the
strip kernel's R = 1 shape for 2D images instead of the row chain
(GEODIST_ROWCHAIN=0)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

VARIANTS = {
    "default": ({}, "any:path=1;any:path=0,rows=4;all:tb=0"),
    "tb": ({"GEODIST_SWEEP_TB": "1"}, "any:tb=1"),
    "rw1": ({"GEODIST_SWEEP_RW": "1"}, "any:rows=4,nwu=4"),
    "rw2": ({"GEODIST_SWEEP_RW": "2"}, "any:kind=2,rows=4,nwu=2"),
    "plane_step": ({"GEODIST_SWEEP_FALLBACK": "1"}, "allp:path=2"),
    "no_cluster": ({"GEODIST_SWEEP_CLUSTER": "0"}, "all:cs=1"),
    "cluster2": ({"GEODIST_SWEEP_CLUSTER": "2"}, "any:cs=2,nwv=1;any:cs=2,nwv=3;none:cs=4"),
    "cluster4": ({"GEODIST_SWEEP_CLUSTER": "4"},
                 "any:cs=4,nwv=1;any:cs=4,nwv=3,kind=1;any:cs=4,kind=0"),
    "cluster8": ({"GEODIST_SWEEP_CLUSTER": "8"}, "any:cs=8,nwv=1;any:cs=8,nwv=3"),
    # the one-row-per-warp (16-warp) shape in clusters of 4: the exact-blend (f64) shape
    "cluster4_rw1": ({"GEODIST_SWEEP_CLUSTER": "4", "GEODIST_SWEEP_RW": "1"},
                     "any:cs=4,rows=4,nwu=4;any:cs=4,nwu=4,kind=2"),
    "no_row_chain": ({"GEODIST_ROWCHAIN": "0"}, "any:path=0,rows=1;none:path=1"),
}


@pytest.mark.parametrize("name", list(VARIANTS))
def test_variant_parity(name):
    env, expect = VARIANTS[name]
    e = dict(os.environ, GD_EXPECT=expect, **env)
    r = subprocess.run([sys.executable, os.path.join(HERE, "_variant_check.py")], env=e,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
