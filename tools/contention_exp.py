"""Experiment: how much does extra HBM traffic on the SMs the 512^3 sweep leaves
free (20 of 148) slow the latency-bound sweep?  Decides whether rotating the
distance between layouts inside the sweep launch (on those SMs) could pay.

python tools/contention_exp.py
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2208_00001_b200 as gd  # noqa: E402


def main():
    L = gd.lib()
    L.gd_debug_background_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_longlong, C.c_int, C.c_int,
                                           C.c_int, C.c_void_p]
    shape = (512, 512, 512)
    img = torch.empty(shape, device="cuda")
    gd.device.fill_splitmix(img, 1)
    mask = torch.ones(shape, device="cuda")
    mask[256, 256, 256] = 0
    out = torch.empty_like(img)
    n = 1 << 28  # 1 GiB
    a = torch.empty(n, device="cuda")
    b = torch.empty(n, device="cuda")
    side = torch.cuda.Stream()

    def run(background, ctas=20, reps=14):
        gd.profile_read(reset=True)
        gd.profile_enable(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        gd.device.generalized_geodesic(img, mask, out, (1, 1, 2.5), 1.0, 1e10, 4)
        if background:
            with torch.cuda.stream(side):
                L.gd_debug_background_copy(a.data_ptr(), b.data_ptr(), n, ctas, 200 * 1024, reps,
                                           side.cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        gd.profile_enable(False)
        prof = gd.profile_read(reset=True)
        return e0.elapsed_time(e1), prof["sweep"][0] / max(prof["sweep"][1], 1)

    for _ in range(2):
        run(False)
    t_bg = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the background copy alone: its bandwidth from 20 CTAs
    t_bg[0].record()
    L.gd_debug_background_copy(a.data_ptr(), b.data_ptr(), n, 20, 200 * 1024, 1, None)
    t_bg[1].record()
    torch.cuda.synchronize()
    ms = t_bg[0].elapsed_time(t_bg[1])
    print(f"background copy alone, 20 CTAs: {ms:.2f} ms for 2 GiB moved -> {2 * n * 4 / ms / 1e6:.0f} GB/s")
    for bg in (False, True, False, True):
        tot, sw = run(bg)
        print(f"background={bg}: transform {tot:.3f} ms, mean sweep launch {sw:.4f} ms")


if __name__ == "__main__":
    main()
