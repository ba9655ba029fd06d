"""The paper's §6 experiment at B200 scale.

PAPER.md:245-300 (§6): FCFS timed against torch.resize for six up-scaling and
six down-scaling factors (2/11 and 27/11 named) x nearest /
bilinear / bicubic on 1024x1024 CelebA images, 100 repeats; plus PSNR / SSIM
between the two outputs.  Here, on one B200:

  * input: a batch of N synthetic 3 x 1024 x 1024 fp32 images (CelebA stand-in,
    not available offline): per channel the seeded smooth field of config 5
    (16 sinusoids + 1% noise) mapped to [0, 1);
  * FCFS: this library (the kernel each plan selects), output floor(1024 p/q);
  * context columns on the same GPU: torch F.interpolate (the comparison
    system; its bilinear/bicubic sample a half-pixel grid with a = -0.75, so the
    values differ by design, reading Z1/Z7) and the paper's own single-layer
    formulation as torch ops (F.pad -> F.conv2d with p^2 output channels per
    channel, stride q -> F.pixel_shuffle, weights = this plan's phase table);
  * times: CUDA events around a CUDA graph of REPS back-to-back launches
    (steady state, inputs larger than L2), per image;
  * image quality (PSNR / SSIM) is measured against the oracle, not against
    F.interpolate: tests/test_gpu_sweep_quality.py (profiles/r02b/sweep_quality.md).

    python tools/paper_sweep.py [--n 16] [--reps 20] [--out profiles/sweep_r01]

Writes <out>.json and <out>.md.  A developer tool: it never touches oracle/.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
from fractions import Fraction

import numpy as np
import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2203_10670_b200 as fc  # noqa: E402

UP = [(27, 11), (2, 1), (7, 4), (5, 3), (3, 2), (4, 3)]
DOWN = [(2, 11), (1, 4), (1, 2), (4, 7), (2, 3), (3, 4)]
MODES = ["nearest", "bilinear", "bicubic"]


def make_images(n: int, size: int = 1024) -> torch.Tensor:
    imgs = np.empty((n, 3, size, size), np.float32)
    for i in range(n):
        for c in range(3):
            v = synth.field_f32(synth.SEED_BASE + 600 + 3 * i + c, size, size, 0, size)
            imgs[i, c] = (v + 1.01) / 2.02  # [-1, 1.01) -> [0, 1)
    return torch.from_numpy(imgs)


def timed(fn, reps: int, stream) -> float:
    """us per call: CUDA graph of reps calls, one replay between events."""
    with torch.cuda.stream(stream):
        fn(0)
        fn(1)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for r in range(reps):
            fn(r)
    with torch.cuda.stream(stream):
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def make_unfused_layer(pl: "fc.Plan", Ho: int, Wo: int, dev):
    """pad -> conv2d (p*p channels per input channel, stride q) -> pixel_shuffle -> crop,
    as a function of x (weights built once, outside any graph capture)."""
    p, q = pl.p, pl.q
    w, base = pl.phase_table()
    T = pl.info.ntaps
    lo = pl.info.lo
    first = [b + lo for b in base]
    wlo = min(first)
    whi = max(f + T - 1 for f in first)
    K = whi - wlo + 1
    k1 = torch.zeros(p, K, dtype=torch.float64)
    for j in range(p):
        if (j * q) % p == 0 or T == 1:  # fraction 0: the tap at offset 0
            k1[j, base[j] - wlo] = 1.0
        else:
            for t in range(T):
                k1[j, first[j] - wlo + t] = w[j][t]
    k2 = torch.einsum("ai,bj->abij", k1, k1).reshape(p * p, 1, K, K).to(torch.float32).to(dev)
    nh, nw = -(-Ho // p), -(-Wo // p)
    H, W = pl.H, pl.W
    pt, pb = -wlo, max(0, (nh - 1) * q + K - H + wlo)
    pleft, pr = -wlo, max(0, (nw - 1) * q + K - W + wlo)
    mode = {"zero": "constant", "replicate": "replicate", "reflect": "reflect"}[pl.pad]

    def layer(x):
        xp = F.pad(x.reshape(-1, 1, H, W), (pleft, pr, pt, pb), mode=mode)
        hid = F.conv2d(xp, k2, stride=q)
        return F.pixel_shuffle(hid, p)[..., :Ho, :Wo].reshape(x.shape[0], x.shape[1], Ho, Wo)
    return layer


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "sweep_r01"))
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    x_host = make_images(args.n)
    xs = [x_host.to(dev), x_host.to(dev)]  # two copies alternate (each > L2)
    rows = []
    for mode in MODES:
        for (p, q) in UP + DOWN:
            r = Fraction(p, q)
            pl = fc.Plan(p, q, mode, "replicate", 3, 1024, 1024, "float32", "floor")
            Ho, Wo = pl.Ho, pl.Wo
            outs = [torch.empty((args.n, 3, Ho, Wo), device=dev) for _ in range(2)]
            kern = pl.launch_info(args.n)["kernel"]
            t_fcfs = timed(lambda i: pl.run(xs[i % 2], out=outs[i % 2], stream=stream), args.reps, stream)
            tmode = {"nearest": "nearest", "bilinear": "bilinear", "bicubic": "bicubic"}[mode]
            kw = {} if mode == "nearest" else {"align_corners": False}
            t_interp = timed(lambda i: F.interpolate(xs[i % 2], size=(Ho, Wo), mode=tmode, **kw), args.reps, stream)
            # the unfused layer materialises the hidden tensor: time it on 2 images
            x2 = [xs[0][:2].contiguous(), xs[1][:2].contiguous()]
            unfused_layer = make_unfused_layer(pl, Ho, Wo, dev)
            try:
                t_unf = timed(lambda i: unfused_layer(x2[i % 2]), max(2, args.reps // 4), stream) / 2
            except torch.OutOfMemoryError:
                t_unf = None
            torch.cuda.synchronize()
            y = pl.run(xs[0][:1])
            yu = unfused_layer(xs[0][:1])
            nbytes = pl.compulsory_bytes(args.n)
            rows.append({
                "mode": mode, "factor": f"{p}/{q}", "scale": float(r), "out": [Ho, Wo], "kernel": kern,
                "fcfs_us_per_image": t_fcfs / args.n, "fcfs_GBps": nbytes / (t_fcfs * 1e-6) / 1e9,
                "interpolate_us_per_image": t_interp / args.n,
                "unfused_layer_us_per_image": t_unf,
                "speedup_vs_interpolate": t_interp / t_fcfs,
                "max_abs_diff_vs_unfused_layer": float((y - yu).abs().max().item()),
            })
            print(json.dumps(rows[-1]), flush=True)
            del outs
            torch.cuda.empty_cache()
    meta = {"gpu": torch.cuda.get_device_name(dev), "batch": args.n, "image": [3, 1024, 1024], "dtype": "float32",
            "reps": args.reps, "pad": "replicate", "extent": "floor",
            "timing": "CUDA events around one CUDA-graph replay of reps back-to-back calls; per image = / batch"}
    with open(args.out + ".json", "w") as f:
        json.dump({"meta": meta, "rows": rows}, f, indent=1)
    with open(args.out + ".md", "w") as f:
        f.write(f"# Paper §6 sweep on B200 (PAPER.md:245-300)\n\n{json.dumps(meta)}\n\n")
        f.write("| mode | factor | out | FCFS kernel | FCFS us/img | FCFS GB/s | F.interpolate us/img | speedup | "
                "unfused layer us/img | max diff vs unfused |\n")
        f.write("|---|---|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            unf = "-" if r["unfused_layer_us_per_image"] is None else f"{r['unfused_layer_us_per_image']:.1f}"
            f.write(f"| {r['mode']} | {r['factor']} | {r['out'][0]}x{r['out'][1]} | {r['kernel']} | "
                    f"{r['fcfs_us_per_image']:.2f} | {r['fcfs_GBps']:.0f} | {r['interpolate_us_per_image']:.2f} | "
                    f"{r['speedup_vs_interpolate']:.2f}x | {unf} | {r['max_abs_diff_vs_unfused_layer']:.2e} |\n")
    print("wrote", args.out + ".json", args.out + ".md")


if __name__ == "__main__":
    main()
