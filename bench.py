#!/usr/bin/env python
"""Benchmark: generalised_geodesic3d, inputs resident in HBM, one process per GPU.

Configs (BASELINE.json):
  * ``--config 512`` (default; the headline): 512^3 float32, spacing
    (1, 1, 2.5), lambda = 1, v = 1e10, it = 4, point-seed soft mask; one volume
    per GPU, so N GPUs = a batch of N independent volumes (weak scaling).
  * ``--config batch64``: the batched config, 64 volumes of 256x256x160 sharded
    by volume across the N ranks (strong scaling: 64 volumes in total); each
    rank runs its shard as one batched transform.
A step = one generalized_geodesic transform (soft-mask init + 24 directional
passes) of every volume this rank owns.  ``value`` = all ranks' voxels / the
max over ranks of the CUDA-event step time (paper_2208_00001_b200.shard.run_sharded);
every working set exceeds the 126 MB L2 (1.5 GB per 512^3 volume; 64 x 40 MB
per batch array), so no flush is needed between steps.  No collective touches
the data path; NCCL carries only the barrier and the timing reduction.

Keys beyond the base contract:
  * ``e2e``: the same transform through the public C-ABI entry
    (gd_generalized_geodesic_batched, GD_MEM_HOST) with pinned host buffers:
    H2D of image + mask and D2H of the distance map inside the timed region.
    512^3: one call over 8 steps' volumes (H2D of step i+1, transform of step i
    and D2H of step i-1 overlap; PCIe H2D-bound); batch64: one call per step;
  * ``roofline``: the directional-pass kernel's algorithmic 12 B/voxel/pass over
    its CUDA-event launch time (events on the launching stream), against
    MEASURED_PEAKS.json hbm_gbs;
  * ``cpu_baseline`` (rank 0, N = 1): the unmodified reference (oracle/_ref) on
    this host's cores, median of 3 after 1 warm-up on the same inputs;
  * ``parity`` (rank 0, any N): the GPU result of rank 0's first volume against
    the reference's on the same inputs, per voxel (1e-6 abs + 1e-5 rel, bit-exact
    fraction).
``--impl reference`` times the reference CPU library alone (rank 0 only) on the
same config: each step one full volume (512) or a 2-volume sample (batch64).
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

NU = 1e10
ITERS = 4
UNIT = "Gvoxels/s"
CONFIGS = {
    "512": dict(shape=(512, 512, 512), spacing=(1.0, 1.0, 2.5), total=None,
                metric="Gvoxels/sec generalised_geodesic3d 512^3 it=4", ref_sample=1),
    "batch64": dict(shape=(256, 256, 160), spacing=(1.0, 1.0, 1.0), total=64,
                    metric="Gvoxels/sec batched generalised_geodesic3d 64 x 256x256x160 it=4",
                    ref_sample=2),
}


def bench_seed(ndim: int, size: int) -> int:
    # tools/main.cpp:312-314
    return 0x67656F64697374 ^ (ndim << 32) ^ size


def volume_seed(cfg: str, b: int) -> int:
    # volume 0 of the 512 config uses the reference CLI's seed; volume b adds b
    size = 512 if cfg == "512" else 256
    return bench_seed(3, size) + b


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
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return ""


def workload_text(cfg, lam, per_gpu):
    c = CONFIGS[cfg]
    d, h, w = c["shape"]
    sp = ",".join(f"{x:g}" for x in c["spacing"])
    if cfg == "512":
        return (f"generalised_geodesic3d {d}x{h}x{w}, spacing ({sp}), lambda={lam:g}, v=1e10, "
                f"it={ITERS}, point seed, one volume per GPU")
    return (f"batched generalised_geodesic3d {c['total']} x {d}x{h}x{w}, spacing ({sp}), "
            f"lambda={lam:g}, v=1e10, it={ITERS}, point seed, sharded by volume")


def run_reference_arm(args, rank):
    """bench.py --impl reference: the unmodified reference on this host's cores,
    on the same config as our arm (full volumes; batch64: a 2-volume sample)."""
    if rank != 0:
        return 0
    from oracle.pyoracle import REF_SO, RefLib
    c = CONFIGS[args.config]
    if not os.path.exists(REF_SO):
        print(json.dumps({"impl": "reference", "unavailable": f"{REF_SO} not built"}))
        return 0
    ref = RefLib()
    cores = os.cpu_count() or 1
    nvol = c["ref_sample"]
    vols = [(host_image(c["shape"], volume_seed(args.config, b)), point_mask_np(c["shape"]))
            for b in range(nvol)]

    def step():
        for img, mask in vols:
            ref.generalized_geodesic(img, mask, c["spacing"], args.lam, NU, ITERS, workers=cores)

    for _ in range(max(args.warmup, 1)):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    vox = nvol * float(np.prod(c["shape"]))
    value = vox / t / 1e9
    sample = (f"{nvol} full volume(s) of the workload per step (same SplitMix64 images, spacing, "
              f"lambda={args.lam:g}, v=1e10, it={ITERS}, point seed); median of {args.steps} "
              f"after {max(args.warmup, 1)} warm-up")
    line = {
        "impl": "reference", "metric": c["metric"], "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "ms_per_step_mean": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "weak" if args.config == "512" else "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (SplitMix64 image on the 2^-24 grid, point-seed soft mask)",
        "config": {"workload": workload_text(args.config, args.lam, c["total"] or 1),
                   "engine": "reference geodist::generalized_geodesic, Engine::Parallel (OpenMP), "
                             "oracle/_ref built from /root/reference with its own flags"},
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
    ap.add_argument("--config", default="512", choices=sorted(CONFIGS))
    ap.add_argument("--lam", type=float, default=1.0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline / parity legs")
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
    from paper_2208_00001_b200.shard import (CudaTimer, max_over_ranks, run_sharded,
                                             volumes_for_rank)

    c = CONFIGS[args.config]
    shape, spacing = c["shape"], c["spacing"]
    torch.cuda.set_device(local)
    gd.device.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    total = c["total"] or world
    mine = list(volumes_for_rank(total, world, rank))
    nv = len(mine)
    batched = nv > 1
    full = (nv,) + shape if batched else shape
    img = torch.empty(full, dtype=torch.float32, device=dev)
    for i, b in enumerate(mine):
        gd.device.fill_splitmix(img[i] if batched else img, volume_seed(args.config, b))
    mask = torch.ones(full, dtype=torch.float32, device=dev)
    for i in range(nv):
        (mask[i] if batched else mask)[tuple(s // 2 for s in shape)] = 0.0
    out = torch.empty_like(img)
    vox_rank = nv * float(np.prod(shape))

    def step():
        gd.device.generalized_geodesic(img, mask, out, spacing, args.lam, NU, ITERS,
                                       batch=nv if batched else None)

    clk = ClockSampler(list(range(max(world, 1)))) if rank == 0 else None
    if clk:
        clk.start()
    marks = {}

    def on_start():
        marks["n0"] = gd.kernel_launches()
        gd.profile_read(reset=True)
        gd.profile_enable(True)
        if clk:
            clk.mark_start()

    def on_end():
        if clk:
            clk.mark_end()
        gd.profile_enable(False)
        marks["prof"] = gd.profile_read(reset=True)
        marks["launches"] = gd.kernel_launches() - marks["n0"]

    res = run_sharded(step, vox_rank, args.steps, args.warmup, timer=CudaTimer(), device=dev,
                      on_start=on_start, on_end=on_end)
    ms, ms_max, value = res["ms_rank"], res["ms_max"], res["gvox_per_s"]
    # stop nvidia-smi before the host-driven legs: its driver queries stall the
    # CUDA API calls the pipelined e2e path issues (measured: 79 vs 25 ms/volume)
    clocks = None
    if clk:
        clk.stop()
        clocks = clk.summary()
    prof, launches = marks["prof"], marks["launches"]

    # ---- roofline of the dominant kernel (the directional-pass sweep) ------
    peak, peak_kind = peak_hbm()
    sw_ms, sw_n, sw_bytes = prof["sweep"]
    achieved = (sw_bytes / sw_n) / (sw_ms / sw_n * 1e-3) / 1e9 if sw_n else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_sweep_traffic.json")
    if os.path.exists(tpath) and args.config == "512":
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak if peak else None, "traffic": traffic,
        "peak_source": f"{peak_kind} MEMORY copy (MEASURED_PEAKS.json hbm_gbs)",
        "kernel": "sweep_kernel (one launch = forward+backward pass pair on one axis)",
        "algorithmic_bytes_per_launch": sw_bytes / sw_n if sw_n else None,
        "bytes_rule": "12 B per voxel per pass (read image, read distance, write distance)",
        "launch_ms": sw_ms / sw_n if sw_n else None,
        "share_of_step": (sw_ms / args.steps) / ms if ms else None,
        "per_class_ms_per_step": {k: v[0] / args.steps for k, v in prof.items()},
        "whole_transform_frac": (12.0 * 6 * ITERS * vox_rank / (ms * 1e-3) / 1e9) / peak,
    }

    # ---- end to end through the C-ABI with pinned host buffers --------------
    # Small steps (one 512^3 volume per rank) are streamed: ONE batched host call
    # over e2e_steps steps' volumes, whose pipeline overlaps step i+1's H2D and
    # step i-1's D2H with step i's transform -- what a caller feeding a stream of
    # volumes gets.  Each step's inputs still cross PCIe inside the timed region.
    # Large steps (the 64-volume batch) are one call per step (pipelined inside).
    import ctypes as C
    step_bytes = 3 * int(vox_rank) * 4
    streamed = step_bytes <= (2 << 30)
    # (8 steps = 12 GiB of pinned host memory per rank at 512^3; 4 when N > 1)
    e2e_steps = args.e2e_steps or min(args.steps, (8 if world == 1 else 4) if streamed else 5)
    reps = e2e_steps if streamed else 1
    while True:  # fewer streamed steps if the host cannot pin that much memory
        hfull = (reps * nv,) + tuple(shape)
        try:
            h_img = torch.empty(hfull, dtype=torch.float32, pin_memory=True)
            h_mask = torch.empty(hfull, dtype=torch.float32, pin_memory=True)
            h_out = torch.empty(hfull, dtype=torch.float32, pin_memory=True)
            break
        except RuntimeError:
            h_img = h_mask = h_out = None
            if reps <= 2:
                raise
            reps //= 2
            e2e_steps = reps
    img_c, mask_c = img.reshape((nv,) + tuple(shape)).cpu(), mask.reshape((nv,) + tuple(shape)).cpu()
    for r in range(reps):
        h_img[r * nv:(r + 1) * nv].copy_(img_c)
        h_mask[r * nv:(r + 1) * nv].copy_(mask_c)
    del img_c, mask_c
    L = gd.lib()
    grid = gd._grid(shape, spacing)

    def e2e_call(nvols):
        rc = L.gd_generalized_geodesic_batched(
            C.byref(grid), nvols, C.c_void_p(h_img.data_ptr()), C.c_void_p(h_mask.data_ptr()),
            args.lam, NU, ITERS, C.c_void_p(h_out.data_ptr()), gd.GD_MEM_HOST, None, None)
        gd._check(rc)

    if streamed:
        e2e_call(min(2, reps) * nv)  # warm-up (untimed)
        e2e_res = run_sharded(lambda: e2e_call(reps * nv), vox_rank * reps, 1, 0,
                              timer=CudaTimer(), device=dev)
        e2e_ms = e2e_res["ms_max"] / reps
        e2e_path = (f"gd_generalized_geodesic_batched(GD_MEM_HOST), pinned host buffers: one call "
                    f"over {reps} steps' volumes, H2D / transform / D2H pipelined across steps")
    else:
        e2e_res = run_sharded(lambda: e2e_call(nv), vox_rank, e2e_steps, 1,
                              timer=CudaTimer(), device=dev)
        e2e_ms = e2e_res["ms_max"]
        e2e_path = ("gd_generalized_geodesic_batched(GD_MEM_HOST), pinned host buffers: one call "
                    "per step, H2D / transform / D2H pipelined over the step's volumes")
    e2e = {"value": e2e_res["gvox_per_s"], "unit": UNIT,
           "h2d_bytes_per_step": 2 * int(vox_rank) * 4, "d2h_bytes_per_step": int(vox_rank) * 4,
           "ms_per_step": e2e_ms, "steps": e2e_steps, "path": e2e_path}
    if streamed:  # one step on its own: H2D, transform, D2H back to back
        lat = run_sharded(lambda: e2e_call(nv), vox_rank, 2, 1, timer=CudaTimer(), device=dev)
        e2e["single_step_latency_ms"] = lat["ms_max"]
    del h_img, h_mask, h_out

    # ---- CPU baseline (reference on this host, N = 1) + parity (rank 0) -----
    cpu_baseline, parity = None, None
    if rank == 0 and not args.no_cpu:
        from oracle.pyoracle import REF_SO, RefLib
        from tests.helpers import parity as parity_fn
        cores = os.cpu_count() or 1
        if os.path.exists(REF_SO):
            ref = RefLib()
            himg = (img[0] if batched else img).cpu().numpy()
            hmask = (mask[0] if batched else mask).cpu().numpy()
            gpu_out = (out[0] if batched else out).cpu().numpy()
            runs = 1 + (3 if world == 1 else 0)  # 1 warm-up + 3 timed, N = 1 only
            times, ref_out = [], None
            for i in range(runs):
                t0 = time.perf_counter()
                ref_out = ref.generalized_geodesic(himg, hmask, spacing, args.lam, NU, ITERS,
                                                   workers=cores)
                if i > 0:
                    times.append(time.perf_counter() - t0)
            if times:
                t_ref = statistics.median(times)
                cpu_baseline = {"value": float(np.prod(shape)) / t_ref / 1e9, "unit": UNIT,
                                "cores": cores, "kind": "reference",
                                "sample": f"one full {'x'.join(map(str, shape))} volume of the "
                                          "workload (same inputs, lambda, it=4), median of 3 "
                                          "after 1 warm-up",
                                "cpu": cpu_info(), "seconds": t_ref,
                                "seconds_all": [round(t, 3) for t in times]}
            ok, exact, max_abs, max_rel = parity_fn(gpu_out, ref_out)
            parity = {"vs": f"reference (oracle/_ref), rank 0 volume {mine[0]}",
                      "within_tolerance": ok, "bit_exact_fraction": exact, "max_abs": max_abs,
                      "max_rel": max_rel, "tolerance": "1e-6 abs + 1e-5 rel, sentinels exact"}
        elif world == 1:
            cpu_baseline = {"value": None, "unit": UNIT, "cores": cores, "kind": "reference",
                            "sample": "unavailable: oracle/_ref not built"}

    launches = int(max_over_ranks(launches, dev))
    if rank == 0:
        line = {
            "metric": c["metric"], "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "weak" if args.config == "512" else "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (SplitMix64 image on the 2^-24 grid, point-seed soft mask)",
            "config": {"workload": workload_text(args.config, args.lam, nv),
                       "volumes_total": total, "volumes_rank0": nv,
                       "l2": "inputs larger than L2 (no flush)",
                       "parallelism": f"volume-sharded x{world}, no collective on the scan"},
            "roofline": roofline, "cpu_baseline": cpu_baseline, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks, "parity": parity,
        }
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
