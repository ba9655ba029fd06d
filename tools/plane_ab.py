"""A/B timing: the plane-resident kernel vs the row-pipelined fused kernel
(FCFS_NO_PLANE) on batches of small planes (developer tool; one GPU).

    python tools/plane_ab.py [--quick]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_10670_b200 import Plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--quick", action="store_true")
a = ap.parse_args()


def time_run(pl, xs, ys, reps=20):
    s = torch.cuda.current_stream()
    for i in range(3):
        pl.run(xs[i % len(xs)], out=ys[i % len(ys)])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for i in range(reps):
        pl.run(xs[i % len(xs)], out=ys[i % len(ys)])
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


pairs = [(5, 3)] if a.quick else [(2, 1), (3, 2), (4, 3), (5, 3), (5, 4), (7, 5), (1, 2), (2, 3), (3, 4), (3, 5), (4, 5), (5, 7)]
shapes = [("bfloat16", 64, 64, 128, 128), ("float16", 32, 64, 96, 96), ("float32", 64, 64, 64, 64), ("bfloat16", 128, 64, 64, 64)]
print("| dtype | N x C x H x W | p/q | mode | plane us | row-pipelined us | plane/row | kernel |")
print("|---|---|---|---|---|---|---|---|")
for dt, N, C, H, W in shapes:
    for (p, q) in pairs:
        for mode in ("bilinear", "bicubic"):
            pl = Plan(p, q, mode, "reflect", C, H, W, dt, "floor")
            kern = pl.launch_info(N)["kernel"]
            esz = torch.finfo(getattr(torch, dt)).bits // 8
            nb = max(2, int(2 * 512e6 // (N * C * (H * W + pl.Ho * pl.Wo) * esz)))
            xs = [torch.randn(N, C, H, W, device="cuda").to(getattr(torch, dt)) for _ in range(nb)]
            ys = [torch.empty(N, C, pl.Ho, pl.Wo, device="cuda", dtype=getattr(torch, dt)) for _ in range(nb)]
            t_plane = time_run(pl, xs, ys) if kern == "fused_plane" else float("nan")
            os.environ["FCFS_NO_PLANE"] = "1"
            t_row = time_run(pl, xs, ys)
            del os.environ["FCFS_NO_PLANE"]
            print(f"| {dt} | {N}x{C}x{H}x{W} | {p}/{q} | {mode} | {t_plane:.1f} | {t_row:.1f} | {t_plane / t_row:.2f} | {kern} |",
                  flush=True)
            del xs, ys
            torch.cuda.empty_cache()
