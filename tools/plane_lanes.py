"""Per-output cost of the plane kernel with 22 vs 32 busy lanes (5/3 bf16 at 64 x 128 / 64 x 192;
developer tool, one GPU): python tools/plane_lanes.py"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2203_10670_b200 import Plan
def t(pl, x, y, reps=20):
    for i in range(3): pl.run(x[i % 2], out=y[i % 2])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps): pl.run(x[i % 2], out=y[i % 2])
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
for (H, W) in [(64, 128), (64, 192), (128, 128), (96, 192)]:
    for mode in ["bicubic", "bilinear"]:
        pl = Plan(5, 3, mode, "reflect", 64, H, W, "bfloat16", "floor")
        info = pl.launch_info(64)
        x = [torch.randn(64, 64, H, W, device="cuda").bfloat16() for _ in range(2)]
        y = [torch.empty(64, 64, pl.Ho, pl.Wo, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
        us = t(pl, x, y)
        nout = 64 * 64 * pl.Ho * pl.Wo
        byts = 2 * 64 * 64 * (H * W + pl.Ho * pl.Wo)
        print(H, W, mode, info["kernel"], info.get("nch"), f"{us:.1f} us", f"{us * 1e3 / nout * 1e3:.3f} ps/out", f"{byts / us / 1e3:.0f} GB/s")
