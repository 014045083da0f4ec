#!/usr/bin/env python
"""Benchmark: generalised_geodesic3d on 512^3, spacing (1,1,2.5), lambda=1, v=1e10, it=4.

Contract:
  * a step = one generalized_geodesic transform (soft-mask init + 24 directional
    passes) of one 512^3 volume per GPU; N GPUs = N independent volumes
    (weak scaling, no collective on the scan);
  * `value` = total voxels / device time (CUDA events, max over ranks), inputs
    resident in HBM; every volume (1.5 GB of image+mask+dist) exceeds the 126 MB
    L2, so no flush is needed between steps;
  * `e2e` = the same transform through the public C-ABI with pinned HOST buffers:
    H2D of image + mask and D2H of the distance map inside the timed region;
  * `roofline` = the directional-pass kernel's algorithmic 12 B/voxel/pass over
    its CUDA-event launch time, against MEASURED_PEAKS.json hbm_gbs;
  * `cpu_baseline` = the unmodified reference (oracle/_ref) on this host's cores,
    also used for a full-size parity check of the GPU result.
`--impl reference` times the reference CPU library alone (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SHAPE = (512, 512, 512)
SPACING = (1.0, 1.0, 2.5)
NU = 1e10
ITERS = 4
METRIC = "Gvoxels/sec generalised_geodesic3d 512^3 it=4"
UNIT = "Gvoxels/s"


def bench_seed(ndim: int, size: int) -> int:
    return 0x67656F64697374 ^ (ndim << 32) ^ size


def volume_seed(b: int) -> int:
    # volume 0 uses the reference CLI's seed (tools/main.cpp:312-314); volume b adds b
    return bench_seed(3, 512) + b


def host_image(shape, seed):
    from oracle.pyoracle import splitmix64_unit
    return splitmix64_unit(int(np.prod(shape)), seed).reshape(shape)


def point_mask_np(shape):
    m = np.ones(shape, np.float32)
    m[tuple(s // 2 for s in shape)] = 0.0
    return m


def peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons, sampled from before the warm-up; the
    summary keeps only the samples inside the timed window (mark_start/mark_end)."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.t0 = self.t1 = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", ",".join(str(g) for g in self.gpus)],
                stdout=self.fh, stderr=subprocess.DEVNULL)
            time.sleep(0.5)  # let the sampler come up before the timed region
        except Exception:
            self.proc = None
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def stop(self):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            self.proc.wait()
            self.fh.close()

    def summary(self):
        if not self.proc:
            return None
        import datetime
        sm, mx, reasons, n_all = [], [], set(), 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                p = [x.strip() for x in line.split(",")]
                if len(p) < 10:
                    continue
                n_all += 1
                try:
                    ts = datetime.datetime.strptime(p[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                    s, m = float(p[2]), float(p[3])
                except ValueError:
                    continue
                if self.t0 is not None and not (self.t0 - 0.05 <= ts <= self.t1 + 0.05):
                    continue
                sm.append(s)
                mx.append(m)
                for n, v in zip(names, p[6:10]):
                    if v.lower() == "active":
                        reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "samples": 0, "reasons": [],
                    "note": f"no sample inside the timed window ({n_all} total)"}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "samples": len(sm),
                "reasons": sorted(reasons)}


def cpu_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return model


def run_reference_arm(args, rank):
    """bench.py --impl reference: the unmodified reference on this host's cores."""
    if rank != 0:
        return 0
    from oracle.pyoracle import REF_SO, RefLib
    if not os.path.exists(REF_SO):
        print(json.dumps({"impl": "reference", "unavailable": f"{REF_SO} not built"}))
        return 0
    ref = RefLib()
    cores = os.cpu_count() or 1
    depth = 128  # bounded sample: a 128-plane slab of the same volume
    img = host_image(SHAPE, volume_seed(0))[:depth].copy()
    mask = point_mask_np(SHAPE)[:depth].copy()
    mask[depth // 2, SHAPE[1] // 2, SHAPE[2] // 2] = 0.0
    for _ in range(args.warmup):
        ref.generalized_geodesic(img, mask, SPACING, args.lam, NU, ITERS, workers=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ref.generalized_geodesic(img, mask, SPACING, args.lam, NU, ITERS, workers=cores)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    vox = img.size
    value = vox / t / 1e9
    sample = (f"{depth}x512x512 slab of the 512^3 workload (same image, spacing, lambda={args.lam}, "
              f"v=1e10, it=4, point seed), mean of {args.steps} after {args.warmup} warm-up")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (SplitMix64 image, point-seed soft mask)",
        "config": {"workload": f"generalised_geodesic3d {depth}x512x512 slab, spacing (1,1,2.5), "
                               f"lambda={args.lam}, v=1e10, it=4",
                   "engine": "reference geodist::generalized_geodesic, Engine::Parallel (OpenMP)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample, "cpu": cpu_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--lam", type=float, default=1.0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline / parity leg")
    ap.add_argument("--e2e-steps", type=int, default=None)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference_arm(args, rank)

    import torch
    import paper_2208_00001_b200 as gd

    torch.cuda.set_device(local)
    gd.device.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()

    dev = torch.device("cuda", local)
    img = torch.empty(SHAPE, dtype=torch.float32, device=dev)
    gd.device.fill_splitmix(img, volume_seed(rank))
    mask = torch.ones(SHAPE, dtype=torch.float32, device=dev)
    mask[tuple(s // 2 for s in SHAPE)] = 0.0
    out = torch.empty_like(img)

    def step():
        gd.device.generalized_geodesic(img, mask, out, SPACING, args.lam, NU, ITERS)

    clk = ClockSampler(list(range(max(world, 1)))) if rank == 0 else None
    if clk:
        clk.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()

    n0 = gd.kernel_launches()
    gd.profile_read(reset=True)
    gd.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier()
    if clk:
        clk.mark_start()
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    if clk:
        clk.mark_end()
    barrier()
    gd.profile_enable(False)
    prof = gd.profile_read(reset=True)
    launches = gd.kernel_launches() - n0
    ms = e0.elapsed_time(e1) / args.steps
    ms_t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if dist is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    vox = float(np.prod(SHAPE))
    value = world * vox / (ms_max * 1e-3) / 1e9

    # ---- roofline of the dominant kernel (the directional-pass sweep) ------
    peak, peak_kind = peak_hbm()
    sw_ms, sw_n, sw_bytes = prof["sweep"]
    achieved = (sw_bytes / sw_n) / (sw_ms / sw_n * 1e-3) / 1e9 if sw_n else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_sweep_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    step_ms_profiled = sum(v[0] for v in prof.values()) / args.steps
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak if peak else None, "traffic": traffic,
        "peak_source": f"{peak_kind} MEMORY copy (MEASURED_PEAKS.json hbm_gbs)",
        "kernel": "sweep_kernel (one launch = forward+backward pass pair on one axis)",
        "algorithmic_bytes_per_launch": sw_bytes / sw_n if sw_n else None,
        "launch_ms": sw_ms / sw_n if sw_n else None,
        "share_of_step": (sw_ms / args.steps) / ms if ms else None,
        "per_class_ms_per_step": {k: v[0] / args.steps for k, v in prof.items()},
        "step_ms_sum_of_launches": step_ms_profiled,
    }

    # ---- end to end through the C-ABI with pinned host buffers --------------
    e2e_steps = args.e2e_steps or min(args.steps, 5)
    h_img = torch.empty(SHAPE, dtype=torch.float32, pin_memory=True)
    h_mask = torch.empty(SHAPE, dtype=torch.float32, pin_memory=True)
    h_out = torch.empty(SHAPE, dtype=torch.float32, pin_memory=True)
    h_img.copy_(img.cpu())
    h_mask.copy_(mask.cpu())
    import ctypes as C
    L = gd.lib()
    grid = gd._grid(SHAPE, SPACING)

    def e2e_step():
        rc = L.gd_generalized_geodesic(C.byref(grid), C.c_void_p(h_img.data_ptr()),
                                       C.c_void_p(h_mask.data_ptr()), args.lam, NU, ITERS,
                                       C.c_void_p(h_out.data_ptr()), gd.GD_MEM_HOST, None, None)
        gd._check(rc)

    e2e_step()
    torch.cuda.synchronize()
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    f1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / e2e_steps
    e2e_ms = f0.elapsed_time(f1) / e2e_steps
    e_t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
    if dist is not None:
        dist.all_reduce(e_t, op=dist.ReduceOp.MAX)
    e2e_ms = float(e_t.item())
    e2e = {"value": world * vox / (e2e_ms * 1e-3) / 1e9, "unit": UNIT,
           "h2d_bytes_per_step": 2 * int(vox) * 4, "d2h_bytes_per_step": int(vox) * 4,
           "ms_per_step": e2e_ms, "wall_ms_per_step": wall * 1e3, "steps": e2e_steps,
           "path": "gd_generalized_geodesic(GD_MEM_HOST) with pinned host buffers"}

    # ---- CPU baseline (reference on this host) + full-size parity -----------
    cpu_baseline, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle.pyoracle import REF_SO, RefLib
        from tests.helpers import parity as parity_fn
        if os.path.exists(REF_SO):
            ref = RefLib()
            cores = os.cpu_count() or 1
            himg = h_img.numpy()
            hmask = h_mask.numpy()
            # the GPU result for exactly these inputs
            gpu_out = out.cpu().numpy()
            t0 = time.perf_counter()
            ref_out = ref.generalized_geodesic(himg, hmask, SPACING, args.lam, NU, ITERS,
                                               workers=cores)
            t_ref = time.perf_counter() - t0
            cpu_baseline = {"value": vox / t_ref / 1e9, "unit": UNIT, "cores": cores,
                            "kind": "reference",
                            "sample": "one full 512^3 transform (same inputs, lambda, it=4), "
                                      "single timed run incl. first-call effects",
                            "cpu": cpu_info(), "seconds": t_ref}
            ok, exact, max_abs, max_rel = parity_fn(gpu_out, ref_out)
            parity = {"vs": "reference (oracle/_ref) at 512^3", "within_tolerance": ok,
                      "bit_exact_fraction": exact, "max_abs": max_abs, "max_rel": max_rel,
                      "tolerance": "1e-6 abs + 1e-5 rel, sentinels exact"}
        else:
            cpu_baseline = {"value": None, "unit": UNIT, "cores": os.cpu_count(),
                            "kind": "reference", "sample": "unavailable: oracle/_ref not built"}

    clocks = None
    if clk:
        clk.stop()
        clocks = clk.summary()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (SplitMix64 image on the 2^-24 grid, point-seed soft mask)",
            "config": {"workload": "generalised_geodesic3d 512x512x512, spacing (1,1,2.5), "
                                   f"lambda={args.lam}, v=1e10, it=4, one volume per GPU",
                       "l2": "inputs larger than L2 (1.5 GB per volume), no flush",
                       "parallelism": f"volume-sharded x{world}"},
            "roofline": roofline, "cpu_baseline": cpu_baseline, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks, "parity": parity,
        }
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
