"""Parity of one kernel variant (selected by environment, read once per process).

Run by tests/test_variants_gpu.py in a subprocess:
    GEODIST_SWEEP_TB=1 GD_EXPECT="any:tb=1" python tests/_variant_check.py
Exits 1 with a message on the first mismatch against the C oracle, or when the
launch log (gd_debug_launch_log) shows the variant the environment asked for
never ran.  GD_EXPECT: ';'-separated clauses "any:key=v" (some launch has it; "any:k1=v1,k2=v2" for
a conjunction), "all:key=v" (every launch of the persistent strip kernel has it), "allp:key=v"
(every launch of any path), "none:key=v" (no launch has it); keys are the
gd_launch_rec fields (path, rows, nwu, cs, tb, ...).
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
    # strip counts divisible by 8 on every axis pair, so clusters of 2/4/8 form:
    # z plane 288x300 (72 strips, 3 warp columns), y/x planes 30 rows (8 strips,
    # partial last strip); z plane 62x100 (16 strips, 1 warp column)
    ((30, 288, 300), (1.0, 1.0, 2.5)),
    ((30, 62, 100), (1.0, 1.3, 1.0)),
    ((45, 300), (1.0, 1.5)),  # 2D: row-chain kernel (or the strip kernel's R = 1 shape)
    ((7, 130), (1.0, 1.0)),
]


def check_expectations(log, spec):
    persist = [r for r in log if r["path"] == 0]
    for clause in filter(None, spec.split(";")):
        mode, kv = clause.split(":", 1)
        want = {k: int(v) for k, v in (x.split("=") for x in kv.split(","))}
        pool = persist if mode == "all" else log
        hits = [r for r in pool if all(r[k] == v for k, v in want.items())]
        if mode == "any" and not hits:
            return f"no launch with {kv}"
        if mode in ("all", "allp") and (not pool or len(hits) != len(pool)):
            bad = [r for r in pool if r not in hits][:3]
            return f"launches without {kv}: {bad}"
        if mode == "none" and hits:
            return f"launches with {kv}: {hits[:3]}"
    return None


def main():
    o = COracle()
    gd.launch_log(reset=True)
    log = []
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
            log += gd.launch_log(reset=True)
    err = check_expectations(log, os.environ.get("GD_EXPECT", ""))
    if err:
        print("variant not exercised:", err)
        return 1
    print(f"ok ({len(log)} launches)")
    return 0


if __name__ == "__main__":
    sys.exit(main())
