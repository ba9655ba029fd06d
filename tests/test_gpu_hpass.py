"""The width-only row kernel (csrc/k_hpass.cu) for 2D layers whose row factor
is 1/1 and for rank-1 plans (every row an independent 1D signal), against the
oracle and, bit for bit, against the row-pipelined fused kernel's identity-row
variant and the reference kernel -- every pair of FCFS_HPASS_PAIRS x mode x
dtype x pad.  Per-dimension factors §4.2; forward layer
PAPER.md:106-116 (§3.1); padding §3; weights §5.2.2-3
(PAPER.md:209-229).
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


def hpass_pairs():
    src = open(PAIRS_H).read()
    m = re.search(r"#define\s+FCFS_HPASS_PAIRS\(Y\)((?:[^\n]*\\\n)*[^\n]*)", src)
    assert m
    return [(int(a), int(b)) for a, b in re.findall(r"Y\((\d+),\s*(\d+)\)", m.group(1))]


def make_x(seed, shape, dtype):
    v = synth.normal_f32(seed, int(np.prod(shape))).reshape(shape)
    return torch.from_numpy(v).to(getattr(torch, dtype))


def _run(x, P, Q, mode, pad, dtype, ext, is1d, monkeypatch, what):
    N, C, H, W = x.shape
    if is1d:
        mk = lambda **kw: Plan(P, Q, mode, pad, C, H, W, dtype, ext, is1d=True, **kw)
    else:
        mk = lambda **kw: Plan.nd((1, P), (1, Q), mode, pad, C, (H, W), dtype, ext, **kw)
    pl = mk()
    info = pl.launch_info(N)
    assert info["kernel"] == "fused_hpass" and (info["PX"], info["QX"]) == (P, Q), (what, info)
    xd = x.to(DEV)
    y = pl.run(xd)
    monkeypatch.setenv("FCFS_NO_HPASS", "1")
    assert pl.launch_info(N)["kernel"] == "fused_separable"
    yf = pl.run(xd)
    monkeypatch.delenv("FCFS_NO_HPASS")
    yr = mk(force_reference=True).run(xd)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.uint8), yf.view(torch.uint8)), f"{what}: != row-pipelined fused kernel"
    assert torch.equal(y.view(torch.uint8), yr.view(torch.uint8)), f"{what}: != reference kernel"
    xr = oracle_input(x)
    if is1d:
        ref = oracle.staged(xr, P, Q, mode, pad, floor_extent=ext == "floor", is1d=True)
    else:
        ref = oracle.staged_nd(xr, [1, P], [1, Q], mode, pad, floor_extent=ext == "floor")
    assert tuple(y.shape) == ref.shape, what
    return compare(y, ref, dtype, mode, float(xr.max() - xr.min()), what, x_absmax=float(np.abs(xr).max()))


@pytest.mark.parametrize("pad", ["zero", "replicate", "reflect"])
def test_hpass_variants_vs_oracle(pad, monkeypatch):
    n_relaxed = 0
    for i, ((P, Q), mode, dtype) in enumerate(itertools.product(hpass_pairs(), MODES, DTYPES)):
        ext = ["floor", "paper"][i % 2]
        W = 8 * Q * max(1, 160 // (8 * Q))  # whole 16-B rows in and out for every dtype
        H = [7, 13, 5][i % 3]
        x = make_x(41000 + i, (2, 3, H, W), dtype)
        n_relaxed += _run(x, P, Q, mode, pad, dtype, ext, i % 4 == 3, monkeypatch,
                          f"hpass {P}/{Q} {mode} {pad} {dtype} W={W}{' 1D' if i % 4 == 3 else ''}")
    print(f"hpass variants ({pad}): {n_relaxed} relaxed elements")


def test_hpass_a1_frames_bitwise():
    """The bench's A1 frames (8 x 3 x 2160 x 3840 fp16, bilinear 3/4 on columns,
    replicate) at full size: every output equal to the fused kernel's, none left
    unwritten (NaN-poisoned output)."""
    x = make_x(42000, (8, 3, 2160, 3840), "float16")
    pl = Plan.nd((1, 3), (1, 4), "bilinear", "replicate", 3, (2160, 3840), "float16", "floor")
    assert pl.launch_info(8)["kernel"] == "fused_hpass"
    xd = x.to(DEV)
    y = torch.full(pl.out_shape(8), float("nan"), dtype=torch.float16, device=DEV)
    pl.run(xd, out=y)
    os.environ["FCFS_NO_HPASS"] = "1"
    try:
        yf = pl.run(xd)
    finally:
        del os.environ["FCFS_NO_HPASS"]
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int16), yf.view(torch.int16))
