"""The height-only row kernel (csrc/k_vpass.cu) for 2D layers whose column
factor is 1/1 (§4.2 per-dimension factors), against the
oracle and, bit for bit, against the row-pipelined fused kernel's identity-
column variant and the reference kernel -- every row pair of the variant
table (FCFS_NONUNIT_PAIRS) x mode x dtype x pad on ragged shapes.  Forward
layer PAPER.md:106-116 (§3.1); padding §3; weights
§5.2.2-3.
"""
import itertools
import os
import re

import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import compare, oracle_input

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2203_10670_b200 import Plan

DEV = "cuda:0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PAIRS_H = os.path.join(ROOT, "paper_2203_10670_b200", "csrc", "fused_pairs.h")
DTYPES = ["float32", "float16", "bfloat16"]
MODES = ["bilinear", "bicubic"]
# (H, W): rows 16-B aligned for every dtype; ragged periods
SHAPES = [(37, 72), (53, 136), (29, 48)]


def row_pairs():
    src = open(PAIRS_H).read()
    m = re.search(r"#define\s+FCFS_NONUNIT_PAIRS\(Y\)((?:[^\n]*\\\n)*[^\n]*)", src)
    assert m
    return [(int(a), int(b)) for a, b in re.findall(r"Y\((\d+),\s*(\d+)\)", m.group(1))]


def make_x(seed, shape, dtype):
    v = synth.normal_f32(seed, int(np.prod(shape))).reshape(shape)
    return torch.from_numpy(v).to(getattr(torch, dtype))


@pytest.mark.parametrize("pad", ["zero", "replicate", "reflect"])
def test_vpass_variants_vs_oracle(pad, monkeypatch):
    n_relaxed = 0
    for i, ((P, Q), mode, dtype) in enumerate(itertools.product(row_pairs(), MODES, DTYPES)):
        ext = ["floor", "paper"][i % 2]
        H, W = SHAPES[i % len(SHAPES)]
        if pad == "reflect" and H * P // Q < 2:
            continue
        x = make_x(31000 + i, (2, 3, H, W), dtype)
        pl = Plan.nd((P, 1), (Q, 1), mode, pad, 3, (H, W), dtype, ext)
        info = pl.launch_info(2)
        assert info["kernel"] == "fused_vpass" and (info["PY"], info["QY"]) == (P, Q), info
        xd = x.to(DEV)
        y = pl.run(xd)
        monkeypatch.setenv("FCFS_NO_VPASS", "1")
        assert pl.launch_info(2)["kernel"] == "fused_separable"
        yf = pl.run(xd)
        monkeypatch.delenv("FCFS_NO_VPASS")
        yr = Plan.nd((P, 1), (Q, 1), mode, pad, 3, (H, W), dtype, ext, force_reference=True).run(xd)
        torch.cuda.synchronize()
        what = f"vpass {P}/{Q} {mode} {pad} {dtype}"
        assert torch.equal(y.view(torch.uint8), yf.view(torch.uint8)), f"{what}: != row-pipelined fused kernel"
        assert torch.equal(y.view(torch.uint8), yr.view(torch.uint8)), f"{what}: != reference kernel"
        xr = oracle_input(x)
        ref = oracle.staged_nd(xr, [P, 1], [Q, 1], mode, pad, floor_extent=ext == "floor")
        assert tuple(y.shape) == ref.shape
        n_relaxed += compare(y, ref, dtype, mode, float(xr.max() - xr.min()), what, x_absmax=float(np.abs(xr).max()))
    print(f"vpass variants ({pad}): {n_relaxed} relaxed elements")


def test_vpass_a2_frames_bitwise():
    """The bench's A2 frames (8 x 3 x 2160 x 3840 fp16, bicubic 5/3 on rows,
    reflect) at full size: every output equal to the fused kernel's, no output
    left unwritten (NaN-poisoned output)."""
    x = make_x(32000, (8, 3, 2160, 3840), "float16")
    pl = Plan.nd((5, 1), (3, 1), "bicubic", "reflect", 3, (2160, 3840), "float16", "floor")
    assert pl.launch_info(8)["kernel"] == "fused_vpass"
    xd = x.to(DEV)
    y = torch.full(pl.out_shape(8), float("nan"), dtype=torch.float16, device=DEV)
    pl.run(xd, out=y)
    os.environ["FCFS_NO_VPASS"] = "1"
    try:
        yf = pl.run(xd)
    finally:
        del os.environ["FCFS_NO_VPASS"]
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int16), yf.view(torch.int16))
