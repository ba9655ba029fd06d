"""SURVEY §8(f) row f2, image quality: the paper's §6 factor sweep
(six up- and six down-scaling factors, 2/11 and 27/11
named at PAPER.md:289-300, x nearest / bilinear / bicubic on 1024 x 1024
images) with PSNR and SSIM of the GPU output measured against the ORACLE
(oracle.staged, the layer of §3.1 in double, pinned in test_oracle_pins.py) --
not against the paper's comparison system, whose sampling grid and cubic
differ by design (readings Z1 and Z7).

Input: one synthetic 3 x 1024 x 1024 fp32 image, per channel the seeded smooth
field of config 5 mapped to [0, 1) (a stand-in for CelebA, which is not
available offline), replicate padding, floor extent.

Bars: nearest bit-exact (PSNR infinite); bilinear / bicubic within
BASELINE.json's fp32 bar (max |gpu - oracle| <= 1e-5 of the input range), which
for data range 1 means PSNR >= 100 dB, and SSIM >= 0.99999.  The measured
table prints with ``pytest -s`` and is written to $FCFS_SWEEP_QUALITY_OUT
(markdown) when that is set (profiles/r02b/sweep_quality.md).
"""
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2203_10670_b200 import Plan

UP = [(27, 11), (2, 1), (7, 4), (5, 3), (3, 2), (4, 3)]
DOWN = [(2, 11), (1, 4), (1, 2), (4, 7), (2, 3), (3, 4)]
MODES = ["nearest", "bilinear", "bicubic"]


def image():
    v = np.stack([synth.field_f32(synth.SEED_BASE + 600 + c, 1024, 1024, 0, 1024) for c in range(3)])
    return ((v + 1.01) / 2.02).astype(np.float32)[None]  # [-1, 1.01) -> [0, 1)


def psnr(a: np.ndarray, ref: np.ndarray) -> float:
    mse = float(np.mean((a.astype(np.float64) - ref) ** 2))
    return math.inf if mse == 0 else 10 * math.log10(1.0 / mse)


def ssim(a: np.ndarray, ref: np.ndarray) -> float:
    """Mean SSIM over channels (Wang et al. 2004): 11 x 11 Gaussian window,
    sigma 1.5, data range 1, K1 = 0.01, K2 = 0.03 -- the paper's metric
    (PAPER.md:276-292).  Evaluated in float64 on the GPU (torch conv2d)."""
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    g = np.exp(-((np.arange(11) - 5.0) ** 2) / (2 * 1.5 ** 2))
    g = torch.from_numpy(g / g.sum()).to(dev)
    gv, gh = g.reshape(1, 1, 11, 1), g.reshape(1, 1, 1, 11)

    def win(t):  # the separable 11 x 11 Gaussian window (valid positions)
        return F.conv2d(F.conv2d(t, gv), gh)

    x = torch.from_numpy(a.astype(np.float64)).reshape(-1, 1, *a.shape[-2:]).to(dev)
    y = torch.from_numpy(ref.astype(np.float64)).reshape(-1, 1, *ref.shape[-2:]).to(dev)
    mx, my = win(x), win(y)
    sxx = win(x * x) - mx ** 2
    syy = win(y * y) - my ** 2
    sxy = win(x * y) - mx * my
    c1, c2 = 0.01 ** 2, 0.03 ** 2
    s = ((2 * mx * my + c1) * (2 * sxy + c2)) / ((mx ** 2 + my ** 2 + c1) * (sxx + syy + c2))
    return float(s.mean())


def test_sweep_psnr_ssim_vs_oracle():
    x = image()
    xd = torch.from_numpy(x).cuda()
    rows = []
    for mode in MODES:
        for p, q in UP + DOWN:
            pl = Plan(p, q, mode, "replicate", 3, 1024, 1024, "float32", "floor")
            y = pl.run(xd)
            torch.cuda.synchronize()
            yg = y.cpu().numpy()
            ref = oracle.staged(x, p, q, mode, "replicate", floor_extent=True)
            assert yg.shape == ref.shape
            err = float(np.abs(yg.astype(np.float64) - ref).max())
            rows.append((mode, f"{p}/{q}", yg.shape[-2:], pl.launch_info(1)["kernel"], err, psnr(yg, ref),
                         ssim(yg, ref)))
            what = f"{mode} {p}/{q}"
            if mode == "nearest":
                np.testing.assert_array_equal(yg.view(np.uint32), ref.astype(np.float32).view(np.uint32), err_msg=what)
            else:
                assert err <= 1e-5 * float(x.max() - x.min()), what
                assert rows[-1][5] >= 100.0 and rows[-1][6] >= 0.99999, (what, rows[-1])
    lines = ["| mode | factor | output | kernel | max abs err vs oracle | PSNR vs oracle (dB) | SSIM vs oracle |",
             "|---|---|---|---|---|---|---|"]
    for mode, f, shp, kern, err, ps, ss in rows:
        lines.append(f"| {mode} | {f} | {shp[0]}x{shp[1]} | {kern} | {err:.2e} | "
                     f"{'inf' if math.isinf(ps) else f'{ps:.1f}'} | {ss:.7f} |")
    table = "\n".join(lines)
    print("\n" + table)
    out = os.environ.get("FCFS_SWEEP_QUALITY_OUT")
    if out:
        with open(out, "w") as f:
            f.write("# Paper §6 factors: FCFS (B200, fp32) vs the oracle, PSNR / SSIM\n\n"
                    "tests/test_gpu_sweep_quality.py: one synthetic 3 x 1024 x 1024 image (config 5's smooth "
                    "field in [0, 1)), replicate padding, floor extent; oracle = oracle.staged (double).\n\n"
                    + table + "\n")
