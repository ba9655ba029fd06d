"""Pins of the oracle's adjoint (backward pass).

FCFS is linear, y = A x; the input gradient is A^T g.  The oracle computes
A^T as the literal transpose of each staged step in reverse order
(oracle.adjoint_nd).  Pinned against what defines an adjoint, not against a
retyped copy of itself:
  * the dot-product identity <A x, g> = <x, A^T g> with the (separately
    pinned) forward oracle, over ranks, factors, modes, pads and extents;
  * the explicit matrix: A built column by column from forward unit impulses,
    then A^T g by numpy;
  * torch float64 autograd through the paper's layer as library ops
    (F.pad -> F.conv2d -> F.pixel_shuffle -> crop), whose backward includes
    torch's own pad adjoints (replicate / reflect accumulation);
  * closed forms: identity, and integer nearest up-scaling whose adjoint is
    sum pooling over p x p blocks.
"""
import itertools

import numpy as np
import pytest

import oracle
import synth

MODES = ["nearest", "bilinear", "bicubic"]
PADS = ["zero", "replicate", "reflect"]


def rng_input(seed, shape):
    return synth.uniform_f32(seed, int(np.prod(shape))).reshape(shape).astype(np.float64) - 0.5


def test_dot_product_identity_sweep():
    rs = np.random.RandomState(51)
    cases = [((9, 11), (3, 5), (2, 3)), ((13,), (2,), (11,)), ((4, 5, 6), (2, 3, 1), (3, 2, 1)),
             ((7, 8), (27, 2), (11, 5)), ((6, 7, 5), (5, 4, 3), (3, 7, 2)), ((17, 19), (4, 4), (7, 7))]
    n = 0
    for (dims, p, q), mode, pad, ext in itertools.product(cases, MODES, PADS, (False, True)):
        x = rng_input(500 + n, (2,) + dims)
        n += 1
        try:
            ax = oracle.staged_nd(x, p, q, mode, pad, floor_extent=ext)
        except oracle.OracleError as e:
            assert e.code in (-2, -3)
            continue
        g = rs.standard_normal(ax.shape)
        atg = oracle.adjoint_nd(g, dims, p, q, mode, pad, floor_extent=ext)
        lhs, rhs = float((ax * g).sum()), float((x * atg).sum())
        assert abs(lhs - rhs) <= 1e-11 * max(1.0, abs(lhs)), (dims, p, q, mode, pad, ext, lhs, rhs)
    assert n == len(cases) * 18


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("pad", PADS)
def test_adjoint_equals_explicit_matrix_transpose(mode, pad):
    for dims, p, q in [((5, 6), (3, 2), (2, 3)), ((4, 3, 5), (2, 3, 5), (3, 2, 4))]:
        nin = int(np.prod(dims))
        try:
            cols = [oracle.staged_nd(np.eye(nin)[k].reshape(dims), p, q, mode, pad).ravel() for k in range(nin)]
        except oracle.OracleError as e:
            assert pad == "reflect" and e.code == -2
            continue
        A = np.stack(cols, axis=1)  # (n_out, n_in)
        odims = oracle.output_dims_nd(dims, p, q, False)
        g = rng_input(61, odims)
        np.testing.assert_allclose(oracle.adjoint_nd(g, dims, p, q, mode, pad).ravel(), A.T @ g.ravel(),
                                   rtol=0, atol=1e-12)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("pad", PADS)
def test_adjoint_equals_torch_autograd_of_the_layer(mode, pad):
    import torch
    import torch.nn.functional as F
    H, W = 19, 23
    for (p, q), ext in itertools.product([(3, 2), (2, 3), (5, 3), (3, 5)], (False, True)):
        x = torch.from_numpy(rng_input(62, (H, W))).requires_grad_(True)
        Ho, Wo = oracle.output_shape(H, W, p, q, ext)
        kers = [oracle.kernel2d(mode, p, q, jy, jx) for jy in range(p) for jx in range(p)]
        T, lo = kers[0][0], kers[0][1]
        wt = torch.from_numpy(np.stack([k[2] for k in kers]))[:, None]
        nhy, nhx = -(-Ho // p), -(-Wo // p)
        padb = (nhy - 1) * q + T - H + lo
        padr = (nhx - 1) * q + T - W + lo
        xt = x[None, None]
        if padb < 0:
            xt = xt[..., : H + padb, :]
            padb = 0
        if padr < 0:
            xt = xt[..., :, : W + padr]
            padr = 0
        tmode = {"zero": "constant", "replicate": "replicate", "reflect": "reflect"}[pad]
        y = F.pixel_shuffle(F.conv2d(F.pad(xt, (-lo, padr, -lo, padb), mode=tmode), wt, stride=q), p)[0, 0, :Ho, :Wo]
        g = torch.from_numpy(rng_input(63, (Ho, Wo)))
        (y * g).sum().backward()
        ours = oracle.adjoint_nd(g.numpy(), (H, W), (p, p), (q, q), mode, pad, floor_extent=ext)
        np.testing.assert_allclose(ours, x.grad.numpy(), rtol=0, atol=1e-12)


def test_closed_forms():
    g = rng_input(64, (3, 12, 15))
    # identity: A = I
    for mode, pad in itertools.product(MODES, PADS):
        assert np.array_equal(oracle.adjoint_nd(g, (12, 15), (1, 1), (1, 1), mode, pad), g)
    # nearest p/1: A repeats each pixel p x p times, A^T sums p x p blocks
    for p in (2, 3):
        gg = rng_input(65, (2, 4 * p, 5 * p))
        want = gg.reshape(2, 4, p, 5, p).sum(axis=(2, 4))
        np.testing.assert_allclose(oracle.adjoint_nd(gg, (4, 5), (p, p), (1, 1), "nearest", "zero"), want,
                                   rtol=0, atol=1e-13)
