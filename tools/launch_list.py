"""Compact a `ncu --metrics gpu__time_duration.sum --csv` launch list into per-kernel totals.

python tools/launch_list.py gpurun_out/launches.csv "title" "command" > profiles/rNN_launches_x.csv
"""
import collections
import csv
import re
import sys

UNIT = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.DictReader(lines))
tot = collections.OrderedDict()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"^(void )?(gdb::)?(<unnamed>::)?", "", r["Kernel Name"])
    name = re.sub(r"\(.*\)$", "", name).replace("(int)", "").replace("(bool)", "")
    us = float(r["Metric Value"].replace(",", "")) * UNIT[r["Metric Unit"]]
    c, t = tot.get(name, (0, 0.0))
    tot[name] = (c + 1, t + us)
allus = sum(t for _, t in tot.values())
print(f"# {sys.argv[2]}")
print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare shares)")
print(f"# command: {sys.argv[3]}")
print("kernel,launches,total_us,mean_us,share")
for n, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{n},{c},{t:.1f},{t / c:.1f},{t / allus:.3f}")
