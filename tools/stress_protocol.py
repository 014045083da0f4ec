"""Inter-CTA halo protocol stress test (compute-sanitizer is closed on this
pool): random grid shapes, spacings, batch sizes and lambdas, each run in
subprocesses under every cluster setting (L2-only links, DSMEM clusters of 2,
4, 8), against the C oracle, bit for bit for lambda in {0, 1}.  Run it with the
protocol-checking build (GD_SWEEP_CHECKS: a halo word tagged beyond the step
being read traps) via GEODIST_LIB=.../libgeodist_b200_checks.so.

python tools/stress_protocol.py [--cases 40] [--seed 1]
"""
import argparse
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

CHILD = r'''
import json, os, sys
sys.path.insert(0, os.environ["GD_ROOT"])
import numpy as np
import paper_2208_00001_b200 as gd
from oracle.pyoracle import COracle
from tests.helpers import bitwise_equal, dyadic_image, parity
cases = json.loads(os.environ["GD_CASES"])
o = COracle()
bad = 0
for c in cases:
    rng = np.random.default_rng(c["seed"])
    shape, B, lam = tuple(c["shape"]), c["batch"], c["lam"]
    imgs = dyadic_image(rng, (B,) + shape)
    masks = np.ones((B,) + shape, np.float32)
    for b in range(B):
        masks[b].reshape(-1)[rng.integers(0, masks[b].size, 2)] = 0.0
    g = gd.generalized_geodesic_batched(imgs, masks, c["sp"], lam, 1e10, c["it"])
    for b in range(B):
        r = o.generalized_geodesic(imgs[b], masks[b], c["sp"], lam, 1e10, c["it"])
        ok = bitwise_equal(g[b], r) if lam in (0.0, 1.0) else parity(g[b], r)[0]
        if not ok:
            bad += 1
            print("MISMATCH", c, b, parity(g[b], r), flush=True)
log = gd.launch_log(reset=True)
print(json.dumps({"bad": bad, "cs": sorted({r["cs"] for r in log})}))
sys.exit(1 if bad else 0)
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=40)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    import random
    rnd = random.Random(a.seed)
    cases = []
    for k in range(a.cases):
        d, h, w = rnd.randint(2, 24), rnd.choice([8, 31, 64, 120, 256, 300]), rnd.randint(3, 600)
        cases.append({"shape": [d, h, w], "batch": rnd.choice([1, 1, 2, 5]),
                      "lam": rnd.choice([0.0, 1.0, 0.6]), "it": rnd.choice([1, 2]),
                      "sp": [rnd.choice([1.0, 2.5]), 1.0, rnd.choice([1.0, 0.7])],
                      "seed": rnd.randint(0, 2**31)})
    total_bad = 0
    for cs in ("0", "2", "4", "8"):
        env = dict(os.environ, GD_ROOT=ROOT, GD_CASES=json.dumps(cases), GEODIST_SWEEP_CLUSTER=cs)
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True,
                           timeout=1800)
        last = (r.stdout.strip().splitlines() or ["{}"])[-1]
        print(f"cluster={cs} rc={r.returncode} {last}", flush=True)
        if r.returncode != 0:
            total_bad += 1
            print(r.stdout[-3000:], r.stderr[-3000:])
    print("protocol stress:", "PASS" if total_bad == 0 else "FAIL", f"({a.cases} cases x 4 cluster settings)")
    return 1 if total_bad else 0


if __name__ == "__main__":
    sys.exit(main())
