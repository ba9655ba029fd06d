"""The slice-ring plane kernel (csrc/plane.cuh fcfs_plane3_kernel) for 3D
volumes of small slices, against the oracle and, bit for bit, against the
row-pipelined 3D fused kernel and the reference kernel -- generated from its
variant table (FCFS_PLANE3_PAIRS in csrc/fused_pairs.h).

A 3D layer scales slices by pz/qz, rows by py/qy and columns by px/qx (§4.2,
PAPER.md:154-167, per-dimension factors); the slice taps combine first
(reference contract: slices, columns, rows), so the three kernels agree bit for
bit.  Padding §3 at the volume's ends remaps the slice
coordinate (reflect / replicate) or reads zeros (zero padding: the TMA box
falls outside the tensor).
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
DTYPES = ["bfloat16", "float16", "float32"]
PADS = ["zero", "replicate", "reflect"]
MODES = ["bilinear", "bicubic"]
# slice factors that run with the row/column pair (3D fused variants take any pz <= 16)
ZF = [(5, 3), (3, 2), (1, 2), (2, 1), (3, 5), (4, 3)]


def plane3_pairs():
    src = open(PAIRS_H).read()
    m = re.search(r"#define\s+FCFS_PLANE3_PAIRS\(Y\)((?:[^\n]*\\\n)*[^\n]*)", src)
    assert m
    return [(int(a), int(b)) for a, b in re.findall(r"Y\((\d+),\s*(\d+)\)", m.group(1))]


def make_x(seed, shape, dtype):
    v = synth.normal_f32(seed, int(np.prod(shape))).reshape(shape)
    return torch.from_numpy(v).to(getattr(torch, dtype))


def run3(x, p, q, mode, pad, dtype, extent, monkeypatch):
    """Slice-ring kernel output and launch info; asserts bitwise equality with the
    row-pipelined 3D kernel (FCFS_NO_PLANE3) and the reference kernel."""
    C, D, H, W = x.shape[1:]
    pl = Plan.nd(p, q, mode, pad, C, (D, H, W), dtype, extent)
    info = pl.launch_info(x.shape[0])
    xd = x.to(DEV)
    y = pl.run(xd)
    monkeypatch.setenv("FCFS_NO_PLANE3", "1")
    yf = pl.run(xd)
    assert pl.launch_info(x.shape[0])["kernel"] == "fused_separable"
    monkeypatch.delenv("FCFS_NO_PLANE3")
    yr = Plan.nd(p, q, mode, pad, C, (D, H, W), dtype, extent, force_reference=True).run(xd)
    torch.cuda.synchronize()
    what = f"{p}/{q} {mode} {pad} {dtype} {tuple(x.shape)}"
    assert torch.equal(y.view(torch.uint8), yf.view(torch.uint8)), f"{what}: plane3 != row-pipelined 3D kernel"
    assert torch.equal(y.view(torch.uint8), yr.view(torch.uint8)), f"{what}: plane3 != reference kernel"
    return y, info


@pytest.mark.parametrize("pad", PADS)
def test_plane3_variants_vs_oracle(pad, monkeypatch):
    """Every compiled pair x mode x dtype on a ragged volume (odd slice counts,
    ragged periods), against the oracle's staged 3D layer."""
    n_relaxed, ran = 0, 0
    for i, ((P, Q), mode, dtype) in enumerate(itertools.product(plane3_pairs(), MODES, DTYPES)):
        ext = ["floor", "paper"][i % 2]
        pz, qz = ZF[i % len(ZF)]
        H, W = [(21, 40), (18, 48), (13, 32)][i % 3]
        D = [7, 9, 6][i % 3]
        pl = Plan.nd((pz, P, P), (qz, Q, Q), mode, pad, 2, (D, H, W), dtype, ext)
        if pl.launch_info(2)["kernel"] != "fused_plane3":
            # f32 bicubic slices may not fit taps + 1 buffers: the row-pipelined kernel runs
            assert dtype == "float32", (P, Q, mode, dtype, pl.launch_info(2))
            continue
        x = make_x(21000 + i, (2, 2, D, H, W), dtype)
        y, info = run3(x, (pz, P, P), (qz, Q, Q), mode, pad, dtype, ext, monkeypatch)
        assert info["kernel"] == "fused_plane3" and (info["PY"], info["QY"]) == (P, Q), info
        xr = oracle_input(x)
        ref = oracle.staged_nd(xr, [pz, P, P], [qz, Q, Q], mode, pad, floor_extent=ext == "floor")
        assert tuple(y.shape) == ref.shape
        n_relaxed += compare(y, ref, dtype, mode, float(xr.max() - xr.min()),
                             f"plane3 {pz}/{qz} {P}/{Q} {mode} {pad} {dtype}", x_absmax=float(np.abs(xr).max()))
        ran += 1
    assert ran >= len(plane3_pairs()) * len(MODES) * 2
    print(f"plane3 variants ({pad}): {ran} runs, {n_relaxed} relaxed elements")


@pytest.mark.parametrize("chunks,grid", [(1, 1), (3, 2), (5, 7)])
def test_plane3_slice_ring_schedules(chunks, grid, monkeypatch):
    """Runs of output slices and grids that make a CTA walk many tasks through the
    slice ring (mbarrier phases wrap, runs cross volumes), ring depth at its
    minimum: the same bits as the default schedule and the oracle."""
    P, Q, pz, qz, mode, pad, dtype = 5, 3, 5, 3, "bicubic", "reflect", "bfloat16"
    x = make_x(22000 + chunks, (3, 2, 11, 20, 32), dtype)
    pl = Plan.nd((pz, P, P), (qz, Q, Q), mode, pad, 2, (11, 20, 32), dtype, "floor")
    xd = x.to(DEV)
    y0 = pl.run(xd)
    monkeypatch.setenv("FCFS_DEBUG_PLANE3_CHUNKS", str(chunks))
    monkeypatch.setenv("FCFS_DEBUG_GRID", str(grid))
    monkeypatch.setenv("FCFS_DEBUG_PLANE3_S", "5")
    info = pl.launch_info(3)
    assert info["kernel"] == "fused_plane3" and info["chunks"] == chunks and info["grid"] == grid and info["S"] == 5, info
    out = torch.full_like(y0, float("nan"))
    pl.run(xd, out=out)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), y0.view(torch.int16)), (chunks, grid)
    xr = oracle_input(x)
    ref = oracle.staged_nd(xr, [pz, P, P], [qz, Q, Q], mode, pad, floor_extent=True)
    compare(out, ref, dtype, mode, float(xr.max() - xr.min()), f"plane3 schedule {chunks}/{grid}",
            x_absmax=float(np.abs(xr).max()))


def test_plane3_v2_bitwise_vs_row_pipelined(monkeypatch):
    """The bench's V2 volume (2 x 8 x 64 x 128^2 bf16, 5/3 tricubic, reflect) at
    full size: the slice-ring kernel by default, every output equal to the
    row-pipelined 3D kernel's."""
    shape = (2, 8, 64, 128, 128)
    x = make_x(23000, shape, "bfloat16")
    pl = Plan.nd((5, 5, 5), (3, 3, 3), "bicubic", "reflect", 8, shape[2:], "bfloat16", "floor")
    assert pl.launch_info(2)["kernel"] == "fused_plane3"
    xd = x.to(DEV)
    y = pl.run(xd)
    monkeypatch.setenv("FCFS_NO_PLANE3", "1")
    yf = pl.run(xd)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int16), yf.view(torch.int16))
