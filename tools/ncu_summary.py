"""Summarise an ncu --set full capture of the sweep kernel (run here, no GPU).

python tools/ncu_summary.py gpurun_out/prof.ncu-rep [voxel_updates_per_launch] > profiles/x.txt

Prints the headline counters, the warp-stall breakdown, the hottest SASS
lines and the executed-instruction mix per voxel update.
"""
import collections
import csv
import io
import re
import subprocess
import sys

RAW = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__block_size", "launch__grid_size", "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    vox = float(sys.argv[2]) if len(sys.argv) > 2 else 2 * 512 ** 3
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, units, vals = raw[0], raw[1], raw[2]
    print("== counters")
    for i, n in enumerate(h):
        if n in RAW:
            print(f"  {n:62s} {vals[i]:>16s} {units[i]}")
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source",
                                           "sass"))))
    hh = rows[1]
    si = hh.index("Warp Stall Sampling (All Samples)")
    src = hh.index("Source")
    ie = hh.index("Instructions Executed")
    reasons = [i for i, n in enumerate(hh) if n.startswith("stall_") and "Not Issued" not in n]
    stall = collections.Counter()
    mix = collections.Counter()
    data, total = [], 0
    for r in rows[2:]:
        try:
            s, n = int(r[si]), int(r[ie])
        except (ValueError, IndexError):
            continue
        data.append(r)
        for i in reasons:
            if r[i]:
                stall[hh[i]] += int(r[i])
        op = re.sub(r"^@!?U?P\w+\s+", "", r[src].strip()).split()[0]
        mix[op] += n
        total += n
    T = sum(stall.values()) or 1
    print(f"== warp instructions executed: {total}  ({total * 32 / vox:.1f} per voxel update)")
    print("== stall reasons (share of samples)")
    for k, v in stall.most_common(10):
        print(f"  {k:28s} {100 * v / T:5.1f}%")
    print("== hottest SASS")
    data.sort(key=lambda r: -int(r[si]))
    for r in data[:15]:
        top = sorted([(int(r[i]) if r[i] else 0, hh[i]) for i in reasons], reverse=True)[:2]
        print(f"  {100 * int(r[si]) / T:5.1f}% {r[src][:64]:64s} {top}")
    print("== instruction mix (per voxel update)")
    for op, n in mix.most_common(24):
        print(f"  {op:24s} {n * 32 / vox:6.2f}")


if __name__ == "__main__":
    main()
