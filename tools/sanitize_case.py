"""Small clustered-sweep cases for compute-sanitizer (one tool per run):

    GEODIST_SWEEP_CLUSTER=4 compute-sanitizer --tool memcheck python tools/sanitize_case.py

Runs the persistent sweep with DSMEM cluster links (the environment picks the
cluster size; default policy clusters planes of >= 64 strips) plus the
tagged-L2 links between clusters, on shapes whose strip counts divide by the
cluster size, and checks every result bit for bit against the C oracle.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2208_00001_b200 as gd  # noqa: E402
from oracle.pyoracle import COracle  # noqa: E402
from tests.helpers import bitwise_equal, dyadic_image, point_mask  # noqa: E402

CASES = [((8, 62, 100), (1.0, 1.0, 2.5)), ((6, 256, 512), (1.0, 1.0, 2.5))]


def main():
    o = COracle()
    gd.launch_log(reset=True)
    bad = 0
    for shape, sp in CASES:
        img = dyadic_image(np.random.default_rng(7), shape)
        m = point_mask(shape)
        for lam in (0.0, 1.0):
            g = gd.generalized_geodesic(img, m, sp, lam, 1e10, 1)
            r = o.generalized_geodesic(img, m, sp, lam, 1e10, 1)
            ok = bitwise_equal(g, r)
            bad += not ok
            print(shape, lam, "ok" if ok else "MISMATCH", flush=True)
    cs = sorted({r["cs"] for r in gd.launch_log(reset=True)})
    print("cluster sizes seen:", cs)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
