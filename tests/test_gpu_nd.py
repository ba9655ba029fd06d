"""GPU parity for per-dimension factors and 3D volumes (§4.2).

The CUDA path (fcfs_plan_nd through the C-ABI) against the ND oracle
(oracle.staged_nd, pinned in test_oracle_nd_pins) at the BASELINE.json bar,
and fused / gather kernels against the reference kernel bitwise (one
arithmetic contract).  Sizes span several fused tiles and ragged tails.
"""
import itertools

import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import compare, oracle_input

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2203_10670_b200 import Plan, scale_nd

DEV = "cuda:0"


def make_x(seed, shape, dtype):
    n = int(np.prod(shape))
    if dtype == "bfloat16":
        v = synth.normal_f32(seed, n)
        return torch.from_numpy(v).to(torch.bfloat16).reshape(shape)
    v = synth.uniform_f32(seed, n)
    t = torch.from_numpy(v).reshape(shape)
    return t.to(torch.float16) if dtype == "float16" else t


def run_nd(x, p, q, mode, pad, extent="floor", force_reference=False):
    dt = {torch.float32: "float32", torch.float16: "float16", torch.bfloat16: "bfloat16"}[x.dtype]
    pl = Plan.nd(p, q, mode, pad, x.shape[1], tuple(x.shape[2:]), dt, extent, force_reference=force_reference)
    y = pl.run(x.to(DEV))
    torch.cuda.synchronize()
    return pl, y


def check(x, p, q, mode, pad, extent="floor", expect_kernel=None):
    dt = {torch.float32: "float32", torch.float16: "float16", torch.bfloat16: "bfloat16"}[x.dtype]
    pl, y = run_nd(x, p, q, mode, pad, extent)
    if expect_kernel:
        assert pl.kernel == expect_kernel, (p, q, pl.kernel)
    xr = oracle_input(x)
    ref = oracle.staged_nd(xr, p, q, mode, pad, floor_extent=extent == "floor")
    assert tuple(y.shape) == ref.shape
    compare(y, ref, dt, mode, float(xr.max() - xr.min()), f"{p}/{q} {mode} {pad} {dt}",
            x_absmax=float(np.abs(xr).max()))
    if pl.kernel != "reference":
        _, yr = run_nd(x, p, q, mode, pad, extent, force_reference=True)
        iv = torch.int32 if dt == "float32" else torch.int16
        assert torch.equal(y.view(iv), yr.view(iv)), f"{p}/{q} {mode} {pad} {dt}: kernels differ"
    return pl


@pytest.mark.parametrize("dtype", ["float32", "float16", "bfloat16"])
@pytest.mark.parametrize("mode", ["bilinear", "bicubic"])
def test_anisotropic_2d_fused_variants(dtype, mode):
    """Width-only and height-only factors run the fused kernel (1/1 in the other dimension)."""
    x = make_x(41, (2, 3, 67, 136), dtype)
    for i, (p, q) in enumerate([((1, 3), (1, 4)), ((1, 7), (1, 5)), ((5, 1), (3, 1)), ((2, 1), (5, 1))]):
        pad = ["zero", "replicate", "reflect"][i % 3]
        check(x, p, q, mode, pad, expect_kernel="fused_separable")


@pytest.mark.parametrize("mode", ["nearest", "bilinear", "bicubic"])
@pytest.mark.parametrize("pad", ["zero", "replicate", "reflect"])
def test_anisotropic_2d_any_factors(mode, pad):
    x = make_x(42, (2, 2, 45, 52), "float32")
    for p, q in [((5, 3), (3, 4)), ((7, 2), (4, 9)), ((3, 11), (2, 27))]:
        check(x, p, q, mode, pad, extent="paper")
        check(x, p, q, mode, pad, extent="floor")


@pytest.mark.parametrize("mode", ["nearest", "bilinear", "bicubic"])
@pytest.mark.parametrize("dtype", ["float32", "float16", "bfloat16"])
def test_volumes_3d(mode, dtype):
    x = make_x(43, (2, 2, 9, 21, 34), dtype)
    for i, (p, q) in enumerate([((3, 2, 5), (2, 3, 3)), ((2, 5, 4), (3, 3, 7)), ((1, 3, 3), (1, 2, 2))]):
        check(x, p, q, mode, ["zero", "replicate", "reflect"][i])


@pytest.mark.parametrize("mode", ["bilinear", "bicubic"])
@pytest.mark.parametrize("dtype", ["float32", "float16", "bfloat16"])
def test_volumes_3d_fused_slice_taps(mode, dtype):
    """3D plans whose slice factor is not 1/1 run the fused variants that combine
    the slice taps in the kernel; bitwise equal to the reference kernel."""
    x = make_x(49, (2, 3, 11, 30, 72), dtype)
    for i, (p, q) in enumerate([((3, 2, 2), (2, 3, 3)), ((5, 3, 3), (7, 2, 2)), ((2, 4, 4), (1, 3, 3)),
                                ((11, 5, 5), (4, 4, 4))]):
        for ext in ("floor", "paper"):
            check(x, p, q, mode, ["zero", "replicate", "reflect"][(i + (ext == "paper")) % 3], extent=ext,
                  expect_kernel="fused_separable")


def test_volume_identity_slice_factor_runs_fused():
    x = make_x(44, (2, 3, 5, 40, 64), "float16")
    pl = check(x, (1, 5, 5), (1, 3, 3), "bicubic", "reflect", expect_kernel="fused_separable")
    assert pl.odims == (5,) + oracle.output_dims_nd((40, 64), (5, 5), (3, 3), True)


@pytest.mark.parametrize("mode", ["nearest", "bilinear", "bicubic"])
def test_rank1(mode):
    x = make_x(45, (3, 4, 1001), "float32")
    for p, q in [(3, 2), (2, 3), (7, 5), (27, 11)]:
        check(x, [p], [q], mode, "replicate")


def test_1d_flag_rows_run_fused_and_match():
    """FCFS_FLAG_1D (rows of an image as independent signals) = rank 1 over every row."""
    x = make_x(46, (2, 3, 37, 96), "float32")
    xd = x.to(DEV)
    for mode, (p, q) in itertools.product(["bilinear", "bicubic"], [(3, 2), (4, 7)]):
        pl = Plan(p, q, mode, "reflect", 3, 37, 96, "float32", "floor", is1d=True)
        assert pl.kernel == "fused_separable"
        y = pl.run(xd)
        ref = oracle.staged(oracle_input(x), p, q, mode, "reflect", floor_extent=True, is1d=True)
        compare(y, ref, "float32", mode, 1.0)
        y1 = Plan.nd([p], [q], mode, "reflect", 3 * 37, (96,), "float32", "floor").run(xd.reshape(2, 3 * 37, 96))
        assert torch.equal(y.reshape(y1.shape), y1)


def test_scale_nd_api_and_edges():
    x = make_x(47, (1, 1, 3, 5, 7), "float32").to(DEV)
    y = scale_nd(x, (2, 3, 5), (3, 2, 3), "bilinear", "zero", "paper")
    assert tuple(y.shape) == (1, 1) + oracle.output_dims_nd((3, 5, 7), (2, 3, 5), (3, 2, 3), False)
    # empty batch
    pl = Plan.nd((2, 3, 5), (3, 2, 3), "bilinear", "zero", 1, (3, 5, 7))
    assert pl.run(torch.empty((0, 1, 3, 5, 7), device=DEV)).shape[0] == 0
    # single-element dimensions
    check(make_x(48, (1, 2, 1, 1, 9), "float32"), (3, 2, 2), (1, 3, 3), "bicubic", "replicate", extent="paper")
