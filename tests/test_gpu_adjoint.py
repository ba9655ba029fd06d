"""GPU parity of the backward pass (fcfs_run_adjoint).

grad_in = A^T grad_out against the oracle's adjoint (tests/
test_oracle_adjoint_pins.py pins it).  Tolerance (reading Z21): the
GPU accumulates in fp32 with one rounding per fma, so per element
|gpu - exact| <= 2^-21 * S, S = |A|^T |g| bounded by max|g| times the product
over dimensions of (max_f sum_t |w_t(f)|) * (ceil(T p/q) + T + 1) (the terms an
input element gathers); 16-bit outputs may add one dtype spacing of the exact
value.  Sizes span ragged tails; every mode/pad; ranks 1-3.
"""
import itertools

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2203_10670_b200 as fc
    from paper_2203_10670_b200 import Plan

DEV = "cuda:0"
WSUM = {"nearest": 1.0, "bilinear": 1.0, "bicubic": 1.25}
TAPS = {"nearest": 1, "bilinear": 2, "bicubic": 4}


def bound(mode, p, q, gmax):
    s = gmax
    for pp, qq in zip(p, q):
        s *= WSUM[mode] * (-(-TAPS[mode] * pp // qq) + TAPS[mode] + 1)
    return 2.0 ** -21 * s


def run_adjoint_case(dims, p, q, mode, pad, dtype, N=2, C=2, extent="floor", seed=0):
    pl = Plan.nd(p, q, mode, pad, C, dims, dtype, extent)
    odims = pl.odims
    gv = synth.normal_f32(seed, N * C * int(np.prod(odims))).reshape((N, C) + tuple(odims))
    g = torch.from_numpy(gv).to(getattr(torch, dtype))
    gi = pl.run_adjoint(g.to(DEV))
    torch.cuda.synchronize()
    ref = oracle.adjoint_nd(g.float().numpy(), dims, p, q, mode, pad, floor_extent=extent == "floor")
    got = gi.cpu().double().numpy()
    tol = bound(mode, p, q, float(np.abs(g.float().numpy()).max()))
    spacing = 0.0  # one dtype spacing of the exact value (16-bit outputs round once)
    if dtype == "float16":
        spacing = np.maximum(np.abs(ref) * 2.0 ** -10, 2.0 ** -24)
    elif dtype == "bfloat16":
        spacing = np.abs(ref) * 2.0 ** -7
    err_ok = np.abs(got - ref) <= tol + spacing
    assert err_ok.all(), (dims, p, q, mode, pad, dtype, float(np.abs(got - ref).max()), tol)
    return pl


@pytest.mark.parametrize("mode", ["nearest", "bilinear", "bicubic"])
@pytest.mark.parametrize("pad", ["zero", "replicate", "reflect"])
def test_adjoint_2d(mode, pad):
    for i, (p, q) in enumerate([(3, 2), (2, 3), (5, 3), (3, 5), (7, 4), (27, 11), (2, 11)]):
        run_adjoint_case((37, 53), (p, p), (q, q), mode, pad, "float32", extent=["floor", "paper"][i % 2], seed=i)


@pytest.mark.parametrize("mode", ["bilinear", "bicubic"])
@pytest.mark.parametrize("dtype", ["float16", "bfloat16"])
def test_adjoint_16bit(mode, dtype):
    run_adjoint_case((41, 64), (5, 5), (3, 3), mode, "reflect", dtype, seed=7)
    run_adjoint_case((41, 64), (4, 4), (7, 7), mode, "replicate", dtype, seed=8)


@pytest.mark.parametrize("mode", ["nearest", "bilinear", "bicubic"])
def test_adjoint_ranks_1_and_3_and_anisotropic(mode):
    run_adjoint_case((101,), (3,), (2,), mode, "replicate", "float32", seed=9)
    run_adjoint_case((7, 9, 11), (3, 2, 5), (2, 3, 3), mode, "zero", "float32", seed=10)
    run_adjoint_case((7, 9, 11), (2, 1, 4), (1, 1, 3), mode, "reflect", "float32", seed=11)
    run_adjoint_case((30, 44), (5, 2), (3, 7), mode, "replicate", "float32", seed=12)


def test_autograd_backward_is_the_adjoint():
    """fc.apply(x, plan) differentiates through the layer: x.grad = A^T g, and
    the dot-product identity <A x, g> = <x, A^T g> holds on the GPU."""
    pl = Plan(5, 3, "bicubic", "reflect", 3, 40, 48, "float32", "floor")
    x = torch.from_numpy(synth.uniform_f32(13, 2 * 3 * 40 * 48).reshape(2, 3, 40, 48)).to(DEV).requires_grad_(True)
    y = fc.apply(x, pl)
    g = torch.from_numpy(synth.normal_f32(14, y.numel()).reshape(y.shape)).to(DEV)
    (y * g).sum().backward()
    assert torch.equal(x.grad, pl.run_adjoint(g))
    lhs = float((y.detach().double() * g.double()).sum())
    rhs = float((x.detach().double() * x.grad.double()).sum())
    assert abs(lhs - rhs) <= 1e-4 * max(1.0, abs(lhs))


def test_adjoint_edges():
    pl = Plan(3, 2, "bilinear", "zero", 1, 5, 7, "float32")
    assert pl.run_adjoint(torch.empty((0, 1, pl.Ho, pl.Wo), device=DEV)).shape == (0, 1, 5, 7)
    run_adjoint_case((1, 1), (3, 3), (2, 2), "bicubic", "replicate", "float32", N=1, C=1, extent="paper", seed=15)
