"""The plane-resident fused kernel (csrc/plane.cuh) against the oracle and,
bit for bit, against the reference and the row-pipelined fused kernels --
generated from its variant table (FCFS_PLANE_PAIRS in csrc/fused_pairs.h).

The kernel serves batches of small 2D planes (BASELINE config 3: 4096 planes
of 128^2 bf16 at 5/3 bicubic).  By default the planner takes it only for at
least 2 x SMs planes; FCFS_DEBUG_PLANE_MIN lowers that bar so that small
ragged batches run it here.  Forward layer: PAPER.md:106-116 (§3.1); padding
§3; weights §5.2.2-3.
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
PADS = ["zero", "replicate", "reflect"]
MODES = ["bilinear", "bicubic"]
# (H, W): rows 16-B aligned for every dtype (the TMA box needs it); ragged periods
SHAPES = [(37, 72), (64, 80), (50, 88), (21, 56)]  # 5/3 output widths 120, 133 | 135, 146, 93 | 95


def plane_pairs():
    src = open(PAIRS_H).read()
    m = re.search(r"#define\s+FCFS_PLANE_PAIRS\(Y\)((?:[^\n]*\\\n)*[^\n]*)", src)
    assert m
    return [(int(a), int(b)) for a, b in re.findall(r"Y\((\d+),\s*(\d+)\)", m.group(1))]


@pytest.fixture
def plane_env(monkeypatch):
    monkeypatch.setenv("FCFS_DEBUG_PLANE_MIN", "1")
    yield monkeypatch


def make_x(seed, shape, dtype):
    v = synth.normal_f32(seed, int(np.prod(shape))).reshape(shape)
    return torch.from_numpy(v).to(getattr(torch, dtype))


def run_three(x, p, q, mode, pad, dtype, extent, env):
    """(plane kernel output, its launch info); asserts bitwise equality with the
    reference kernel and the row-pipelined fused kernel."""
    C, H, W = x.shape[1:]
    pl = Plan(p, q, mode, pad, C, H, W, dtype, extent)
    info = pl.launch_info(x.shape[0])
    xd = x.to(DEV)
    y = pl.run(xd)
    yr = Plan(p, q, mode, pad, C, H, W, dtype, extent, force_reference=True).run(xd)
    env.setenv("FCFS_NO_PLANE", "1")
    yf = pl.run(xd)
    assert pl.launch_info(x.shape[0])["kernel"] == "fused_separable"
    env.delenv("FCFS_NO_PLANE")
    torch.cuda.synchronize()
    what = f"{p}/{q} {mode} {pad} {dtype} {tuple(x.shape)}"
    assert torch.equal(y.view(torch.uint8), yr.view(torch.uint8)), f"{what}: plane != reference kernel"
    assert torch.equal(y.view(torch.uint8), yf.view(torch.uint8)), f"{what}: plane != row-pipelined fused kernel"
    return y, info


@pytest.mark.parametrize("pad", PADS)
def test_plane_variants_vs_oracle(pad, plane_env):
    n_relaxed = 0
    for i, ((P, Q), mode, dtype) in enumerate(itertools.product(plane_pairs(), MODES, DTYPES)):
        ext = ["floor", "paper"][i % 2]
        # the first shape (rotating) whose output row fits the kernel's 32 chunks
        for k in range(len(SHAPES) + 1):
            H, W = (SHAPES[(i + k) % len(SHAPES)] if k < len(SHAPES) else (19, 24))
            if Plan(P, Q, mode, pad, 5, H, W, dtype, ext).launch_info(3)["kernel"] == "fused_plane":
                break
        x = make_x(11000 + i, (3, 5, H, W), dtype)
        y, info = run_three(x, P, Q, mode, pad, dtype, ext, plane_env)
        assert info["kernel"] == "fused_plane" and (info["PY"], info["QY"]) == (P, Q), info
        xr = oracle_input(x)
        ref = oracle.staged_nd(xr, [P, P], [Q, Q], mode, pad, floor_extent=ext == "floor")
        n_relaxed += compare(y, ref, dtype, mode, float(xr.max() - xr.min()), f"plane {P}/{Q} {mode} {pad} {dtype}",
                             x_absmax=float(np.abs(xr).max()))
    print(f"plane variants ({pad}): {n_relaxed} relaxed elements")


def test_plane_many_planes_per_cta(plane_env):
    """A small grid: every CTA walks many planes through both plane buffers
    (mbarrier phases wrap several times), bands rotate over the warps."""
    plane_env.setenv("FCFS_DEBUG_GRID", "3")
    for i, (mode, dtype, pad) in enumerate([("bicubic", "bfloat16", "reflect"), ("bilinear", "float16", "replicate"),
                                            ("bicubic", "float32", "zero")]):
        P, Q = [(5, 3), (3, 2), (4, 3)][i]
        x = make_x(12000 + i, (4, 7, 37, 72), dtype)
        y, info = run_three(x, P, Q, mode, pad, dtype, "floor", plane_env)
        assert info["kernel"] == "fused_plane" and info["grid"] == 3, info
        xr = oracle_input(x)
        ref = oracle.staged_nd(xr, [P, P], [Q, Q], mode, pad, floor_extent=True)
        compare(y, ref, dtype, mode, float(xr.max() - xr.min()), f"grid-3 {P}/{Q} {mode} {pad} {dtype}",
                x_absmax=float(np.abs(xr).max()))


def test_plane_c3_bitwise_vs_row_pipelined():
    """BASELINE config 3 (64 x 64 x 128^2 bf16, bicubic 5/3, reflect, floor
    extent 213^2) at full size takes the plane kernel by default; every output
    equals the row-pipelined fused kernel's (whose every output the C3 parity
    test compares with the oracle)."""
    x = synth.make_input(synth.CONFIGS["C3"])
    pl = Plan(5, 3, "bicubic", "reflect", 64, 128, 128, "bfloat16", "floor")
    assert pl.launch_info(64)["kernel"] == "fused_plane"
    xd = x.to(DEV)
    y = pl.run(xd)
    os.environ["FCFS_NO_PLANE"] = "1"
    try:
        yf = pl.run(xd)
    finally:
        del os.environ["FCFS_NO_PLANE"]
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.uint8), yf.view(torch.uint8))
