"""GPU parity of the weight gradient (fcfs_run_weight_grad, SURVEY.md §8(f)
row f3, reading Z22) against the oracle's literal backward of the staged layer
(tests/test_oracle_wgrad_pins.py pins it to torch float64 autograd).

Bar (Z22): every weight is a sum of n products g * x~ (n = the
outputs of its phase pair over all planes), accumulated in fp32 in some order
(register chains, a shared-memory sum, atomics); any such order is within
n * 2^-24 * sum |g| |x~| of the exact value (first order), so the test
requires |gpu - exact| <= (n + 8) * 2^-24 * abs_sum.  16-bit inputs convert
to fp32 exactly; the oracle reads the same dtype values.
"""
import itertools

import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import oracle_input

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2203_10670_b200 as fc
    from paper_2203_10670_b200 import Plan
    from paper_2203_10670_b200._lib import FcfsError

DEV = "cuda:0"


def run_case(N, C, H, W, p, q, mode, pad, dtype, extent="floor", is1d=False, seed=0):
    pl = Plan(p, q, mode, pad, C, H, W, dtype, extent, is1d)
    x = torch.from_numpy(synth.normal_f32(seed, N * C * H * W).reshape(N, C, H, W)).to(getattr(torch, dtype))
    oshape = pl.out_shape(N)
    g = torch.from_numpy(synth.normal_f32(seed + 1, int(np.prod(oshape))).reshape(oshape)).to(getattr(torch, dtype))
    gw = pl.run_weight_grad(x.to(DEV), g.to(DEV))
    torch.cuda.synchronize()
    ref, ab = oracle.weight_grad(oracle_input(x), g.double().numpy(), p, q, mode, pad,
                                 floor_extent=extent == "floor", is1d=is1d)
    assert tuple(gw.shape) == ref.shape
    n = N * C * oshape[-2] * oshape[-1]  # >= the terms of any one weight
    tol = (n + 8) * 2.0 ** -24 * ab + 1e-30
    err = np.abs(gw.cpu().double().numpy() - ref)
    assert (err <= tol).all(), (p, q, mode, pad, dtype, float(err.max()), float(tol.max()))
    return pl, gw


@pytest.mark.parametrize("mode", ["nearest", "bilinear", "bicubic"])
@pytest.mark.parametrize("pad", ["zero", "replicate", "reflect"])
def test_weight_grad_2d(mode, pad):
    for i, ((p, q), dtype) in enumerate(itertools.product([(3, 2), (2, 3), (5, 3), (3, 5), (7, 4), (4, 1), (6, 1)],
                                                          ["float32", "bfloat16"])):
        run_case(2, 3, 29, 45, p, q, mode, pad, dtype, extent=["floor", "paper"][i % 2], seed=10 + i)


@pytest.mark.parametrize("mode", ["bilinear", "bicubic"])
def test_weight_grad_1d_f16_and_large_factors(mode):
    run_case(2, 3, 5, 101, 5, 3, mode, "reflect", "float16", is1d=True, seed=3)
    run_case(1, 2, 33, 70, 27, 11, mode, "replicate", "float32", seed=4)  # 729 phase pairs: 23 lane groups
    run_case(1, 1, 40, 300, 2, 11, mode, "zero", "float32", seed=5)


def test_weight_grad_medium_bf16():
    """C3's factor and layout at 4 x 8 planes: several CTAs, column and row bands."""
    run_case(4, 8, 128, 128, 5, 3, "bicubic", "reflect", "bfloat16", seed=6)


def test_weight_grad_edges():
    pl = Plan(3, 2, "bilinear", "zero", 2, 9, 10, "float32")
    x = torch.empty((0, 2, 9, 10), device=DEV)
    g = torch.empty((0, 2) + tuple(pl.out_shape(1)[2:]), device=DEV)
    gw = pl.run_weight_grad(x, g)
    assert gw.shape == (3, 3, 2, 2) and not gw.any()
    run_case(1, 1, 1, 1, 3, 2, "bicubic", "replicate", "float32", extent="paper", seed=7)
    pl3 = Plan.nd((2, 2, 2), (1, 1, 1), "bilinear", "zero", 1, (3, 4, 5), "float32")
    with pytest.raises(FcfsError) as e:
        pl3.weight_grad_shape()
    assert e.value.name == "FCFS_E_UNSUPPORTED"


def test_weight_grad_is_the_derivative():
    """Finite differences through a forward with perturbed weights are not
    available (the forward has fixed taps), so check the chain rule the other
    way: for nearest 4/1 every output copies one input, and sum(y * g) is
    linear in the weights with coefficient grad_w -- perturbing the (only) tap
    of phase (jy, jx) by e changes sum(y*g) by e * grad_w[jy, jx]."""
    pl = Plan(4, 1, "nearest", "zero", 3, 6, 7, "float32")
    x = torch.from_numpy(synth.normal_f32(8, 2 * 3 * 6 * 7).reshape(2, 3, 6, 7)).to(DEV)
    y = pl.run(x)
    g = torch.from_numpy(synth.normal_f32(9, y.numel()).reshape(y.shape)).to(DEV)
    gw = pl.run_weight_grad(x, g)
    for jy, jx in [(0, 0), (1, 3), (3, 2)]:
        ys = y.clone()
        ys[:, :, jy::4, jx::4] *= 1.5  # weight 1 -> 1.5 for that phase pair
        d = float(((ys - y) * g).double().sum())
        assert abs(d - 0.5 * float(gw[jy, jx, 0, 0])) <= 1e-4 * max(1.0, abs(d))


@pytest.mark.parametrize("dtype", ["float32", "bfloat16", "float16"])
def test_weight_grad_exact_on_integer_inputs(dtype):
    """Integer inputs in [-3, 3]: every product and every partial sum is an
    integer below 2^24, so fp32 accumulation is exact in any order and the GPU
    must equal the oracle exactly -- a pin on the reduction's completeness
    (every plane, period and phase pair counted once) that an error bound
    cannot give at this size."""
    for (N, C, H, W, p, q, mode, pad) in [(4, 8, 128, 128, 5, 3, "bicubic", "reflect"),
                                          (3, 5, 70, 90, 3, 4, "bilinear", "replicate"),
                                          (2, 4, 64, 200, 2, 3, "nearest", "zero")]:
        pl = Plan(p, q, mode, pad, C, H, W, dtype, "floor")
        oshape = pl.out_shape(N)
        xi = np.floor(synth.uniform_f32(21, N * C * H * W) * 7.0) - 3.0
        gi = np.floor(synth.uniform_f32(22, int(np.prod(oshape))) * 7.0) - 3.0
        x = torch.from_numpy(xi.reshape(N, C, H, W).astype(np.float32)).to(getattr(torch, dtype))
        g = torch.from_numpy(gi.reshape(oshape).astype(np.float32)).to(getattr(torch, dtype))
        # bicubic taps are not integers: take the gradient only (it does not use the weights)
        gw = pl.run_weight_grad(x.to(DEV), g.to(DEV))
        torch.cuda.synchronize()
        ref, ab = oracle.weight_grad(oracle_input(x), g.double().numpy(), p, q, mode, pad, floor_extent=True)
        assert ab.max() < 2 ** 24
        assert np.array_equal(gw.cpu().double().numpy(), ref), (p, q, mode, pad, dtype)


def test_kernel_launch_counter():
    """fcfs_kernel_launches counts the library's kernels (the bench's gpu_launches):
    one per forward run, one per weight gradient, two for a replicate-padded 2D
    adjoint (fused interior + border bands)."""
    pl = Plan(5, 3, "bicubic", "replicate", 2, 40, 48, "float32", "floor")
    x = torch.from_numpy(synth.normal_f32(30, 2 * 2 * 40 * 48).reshape(2, 2, 40, 48)).to(DEV)
    n0 = fc.kernel_launches()
    y = pl.run(x)
    assert fc.kernel_launches() - n0 == 1
    n0 = fc.kernel_launches()
    pl.run_weight_grad(x, y)
    assert fc.kernel_launches() - n0 == 1
    n0 = fc.kernel_launches()
    pl.run_adjoint(y)
    assert fc.kernel_launches() - n0 == 2
    torch.cuda.synchronize()


def test_weight_grad_rank1_plan_equals_1d_rows():
    """A rank-1 plan (plan_nd with one factor) has the 1D flag's weights (1, p, 1, taps)."""
    for mode in ("bilinear", "bicubic"):
        pl = Plan.nd((5,), (3,), mode, "reflect", 3, (97,), "float32", "floor")
        assert pl.weight_grad_shape() == (1, 5, 1, {"bilinear": 2, "bicubic": 4}[mode])
        x = torch.from_numpy(synth.normal_f32(40, 2 * 3 * 97).reshape(2, 3, 97))
        g = torch.from_numpy(synth.normal_f32(41, 2 * 3 * pl.odims[0]).reshape(2, 3, pl.odims[0]))
        gw = pl.run_weight_grad(x.to(DEV), g.to(DEV))
        ref, ab = oracle.weight_grad(x.numpy()[:, :, None, :], g.double().numpy()[:, :, None, :], 5, 3, mode, "reflect",
                                     floor_extent=True, is1d=True)
        n = g.numel()
        assert (np.abs(gw.cpu().double().numpy() - ref) <= (n + 8) * 2.0 ** -24 * ab + 1e-30).all()


@pytest.mark.parametrize("mode", ["nearest", "bilinear", "bicubic"])
def test_weight_grad_anisotropic(mode):
    """Per-dimension factors (plan_nd, §4.2): the GPU's anisotropic weight
    gradient against the oracle's (pinned to torch autograd with stride (qy, qx))."""
    for i, (p, q, pad, dtype) in enumerate([((5, 2), (3, 7), "replicate", "float32"),
                                            ((3, 4), (2, 3), "reflect", "bfloat16"),
                                            ((2, 7), (5, 4), "zero", "float32")]):
        H, W = 41, 66
        pl = Plan.nd(p, q, mode, pad, 3, (H, W), dtype, "floor")
        x = torch.from_numpy(synth.normal_f32(60 + i, 2 * 3 * H * W).reshape(2, 3, H, W)).to(getattr(torch, dtype))
        oshape = pl.out_shape(2)
        g = torch.from_numpy(synth.normal_f32(70 + i, int(np.prod(oshape))).reshape(oshape)).to(getattr(torch, dtype))
        gw = pl.run_weight_grad(x.to(DEV), g.to(DEV))
        torch.cuda.synchronize()
        ref, ab = oracle.weight_grad_2d(oracle_input(x), g.double().numpy(), p, q, mode, pad, floor_extent=True)
        assert tuple(gw.shape) == ref.shape, (gw.shape, ref.shape)
        tol = (g.numel() + 8) * 2.0 ** -24 * ab + 1e-30
        assert (np.abs(gw.cpu().double().numpy() - ref) <= tol).all(), (p, q, mode, pad, dtype)


@pytest.mark.parametrize("pad", ["zero", "replicate", "reflect"])
def test_weight_grad_tensor_core_every_compiled_factor(pad, monkeypatch):
    """The tensor-core kernel (16-bit inputs, 16-B aligned rows, the compiled
    factors of FCFS_WG_ROWS in csrc/k_wgrad.cu) on ragged shapes -- output rows
    not a multiple of the band or period, a row's last 16-period block partly
    past the width (masked A fragments), margins of every padding mode from the
    TMA box -- against the oracle at Z22's bound, and exactly on integer
    inputs; fcfs_last_launch asserts the kernel that ran."""
    cases = [(5, 3), (3, 2), (2, 3), (3, 5)]
    for i, ((p, q), mode, dtype) in enumerate(itertools.product(cases, ["bilinear", "bicubic"],
                                                                 ["bfloat16", "float16"])):
        H, W = [(37, 72), (101, 64), (53, 136)][i % 3]
        run_case(2, 3, H, W, p, q, mode, pad, dtype, extent=["floor", "paper"][i % 2], seed=40 + i)
        assert fc.last_launch()["kernel"] == "weight_grad_tensor_core", (p, q, mode, dtype, fc.last_launch())
    # integers: exact in any summation order; 2 and the default (4) tile buffers, many
    # tasks per CTA (every buffer's mbarrier phase wraps)
    pl = Plan(5, 3, "bicubic", pad, 3, 141, 80, "bfloat16", "floor")
    oshape = pl.out_shape(40)
    xi = np.floor(synth.uniform_f32(31, 40 * 3 * 141 * 80) * 7.0) - 3.0
    gi = np.floor(synth.uniform_f32(32, int(np.prod(oshape))) * 7.0) - 3.0
    x = torch.from_numpy(xi.reshape(40, 3, 141, 80).astype(np.float32)).to(torch.bfloat16)
    g = torch.from_numpy(gi.reshape(oshape).astype(np.float32)).to(torch.bfloat16)
    ref, _ = oracle.weight_grad(oracle_input(x), g.double().numpy(), 5, 3, "bicubic", pad, floor_extent=True)
    for nbuf in ("2", None):
        if nbuf:
            monkeypatch.setenv("FCFS_DEBUG_WG_NBUF", nbuf)
        else:
            monkeypatch.delenv("FCFS_DEBUG_WG_NBUF", raising=False)
        gw = pl.run_weight_grad(x.to(DEV), g.to(DEV))
        torch.cuda.synchronize()
        info = fc.last_launch()
        assert info["kernel"] == "weight_grad_tensor_core" and (nbuf is None or info["buffers"] == 2), info
        assert np.array_equal(gw.cpu().double().numpy(), ref), info
