"""Kernel variants reachable only through tuning switches (read once per process),
checked in a subprocess against the C oracle: temporal blocking over plane pairs
(GEODIST_SWEEP_TB=1), the one-row-per-warp strip shape for every cost kind
(GEODIST_SWEEP_RW=1), the two-rows-per-warp shape for blend (RW=2) and the
plane-step fallback for every plane (GEODIST_SWEEP_FALLBACK=1) and DSMEM halo
links inside thread-block clusters (GEODIST_SWEEP_CLUSTER=<cs>), and the strip
kernel's R = 1 shape for 2D images instead of the row chain (GEODIST_ROWCHAIN=0)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("env", [{"GEODIST_SWEEP_TB": "1"}, {"GEODIST_SWEEP_RW": "1"},
                                 {"GEODIST_SWEEP_RW": "2"}, {"GEODIST_SWEEP_FALLBACK": "1"},
                                 {"GEODIST_SWEEP_CLUSTER": "0"}, {"GEODIST_SWEEP_CLUSTER": "2"},
                                 {"GEODIST_SWEEP_CLUSTER": "8"},
                                 {"GEODIST_SWEEP_CLUSTER": "4", "GEODIST_SWEEP_RW": "1"},
                                 {"GEODIST_ROWCHAIN": "0"}],
                         ids=["tb", "rw1", "rw2", "plane_step", "no_cluster", "cluster2",
                              "cluster8", "cluster4_rw1", "no_row_chain"])
def test_variant_parity(env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, os.path.join(HERE, "_variant_check.py")], env=e,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
