"""Parity of one kernel variant (selected by environment, read once per process).

Run by tests/test_variants_gpu.py in a subprocess:
    GEODIST_SWEEP_TB=1 python tests/_variant_check.py
Exits 1 with a message on the first mismatch against the C oracle.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2208_00001_b200 as gd  # noqa: E402
from oracle.pyoracle import COracle  # noqa: E402
from tests.helpers import bitwise_equal, dyadic_image, parity, seed_init  # noqa: E402

CASES = [
    ((37, 53, 41), (1.0, 1.3, 0.7)),
    ((20, 70, 132), (1.0, 1.0, 2.5)),
    ((9, 130, 260), (1.0, 1.0, 1.0)),
    ((24, 17, 520), (2.0, 1.0, 1.0)),
    ((45, 300), (1.0, 1.5)),  # 2D: row-chain kernel (or the strip kernel's R = 1 shape)
    ((7, 130), (1.0, 1.0)),
]


def main():
    o = COracle()
    for shape, sp in CASES:
        for lam in (0.0, 0.7, 1.0):
            rng = np.random.default_rng(hash((shape, lam)) % 2**32)
            img = dyadic_image(rng, shape)
            d0 = seed_init(rng, shape, 4)
            for it in (1, 2):
                g = gd.parallel_scan(img, d0, sp, lam, it)
                r = o.parallel_scan(img, d0, sp, lam, it)
                if lam in (0.0, 1.0):
                    ok = bitwise_equal(g, r)
                else:
                    ok = parity(g, r)[0]
                if not ok:
                    print(f"mismatch shape={shape} lam={lam} it={it}: {parity(g, r)}")
                    return 1
            # single directional passes (npass = 1: no backward half)
            for axis in (range(3) if len(shape) == 3 else (1, 2)):
                for orient in (+1, -1):
                    g = gd.directional_pass(d0, img, axis, orient, sp, lam)
                    r = o.directional_pass(d0, img, axis, orient, sp, lam)
                    ok = bitwise_equal(g, r) if lam in (0.0, 1.0) else parity(g, r)[0]
                    if not ok:
                        print(f"mismatch pass shape={shape} lam={lam} axis={axis} o={orient}")
                        return 1
    print("ok")
    return 0


if __name__ == "__main__":
    sys.exit(main())
