"""Stall-reason totals per code region (split at BAR.SYNC / EXIT) of an ncu source page.

ncu -i rep --page source --csv --print-source sass > src.csv; python tools/ncu_regions.py src.csv
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
regs, cur = [], None
for k, r in enumerate(data):
    if cur is None:
        cur = {"start": r[0][-5:], "s": 0.0, "e": 0.0, "st": [0.0] * len(stalls), "n": 0}
    cur["s"] += float(r[iS] or 0)
    cur["e"] += float(r[iE] or 0)
    cur["n"] += 1
    for j, i in enumerate(stalls):
        cur["st"][j] += float(r[i] or 0)
    if "BAR.SYNC" in r[1] or "EXIT" in r[1] or k == len(data) - 1:
        cur["end"] = r[0][-5:]
        regs.append(cur)
        cur = None
for c in regs:
    if c["s"] < 50:
        continue
    top = sorted(zip(c["st"], [hdr[i][6:] for i in stalls]), reverse=True)[:6]
    print(f"{c['start']}..{c['end']} n={c['n']:4d} inst={c['e']:10.0f} samples={c['s']:6.0f}  " +
          " ".join(f"{n}={v:.0f}" for v, n in top))
