"""Pins of the oracle's weight gradient (reading Z22).

The learnable parameters of output channel (jy, jx) are its own taps (the
nonzero support of the fixed §5.2 kernel); oracle.weight_grad returns
d(sum y*g)/dW over them, summed over planes.  Pinned against what defines it:
  * torch float64 autograd through the paper's layer as library ops
    (F.pad -> F.conv2d with a (p^2, 1, T, T) weight that requires grad ->
    F.pixel_shuffle -> crop), its weight.grad read at each phase's taps;
  * closed forms: nearest p/1 is sum over blocks of g * x[i] per phase; the
    identity 1/1 is the correlation sum g[m] x~[m + t];
  * linearity in g.
"""
import itertools

import numpy as np
import pytest

import oracle
import synth

MODES = ["nearest", "bilinear", "bicubic"]
PADS = ["zero", "replicate", "reflect"]


def rnd(seed, shape):
    return synth.uniform_f32(seed, int(np.prod(shape))).reshape(shape).astype(np.float64) - 0.5


def torch_layer_wgrad(x, g, p, q, mode, pad, ext, is1d=False):
    import torch
    import torch.nn.functional as F
    N, H, W = x.shape
    Ho, Wo = oracle.output_shape(H, W, p, q, ext, is1d)
    kers = [oracle.kernel2d(mode, p, q, jy, jx) for jy in range(p) for jx in range(p)]
    T, lo = kers[0][0], kers[0][1]
    w = torch.from_numpy(np.stack([k[2] for k in kers]))[:, None].clone().requires_grad_(True)
    nhy, nhx = -(-Ho // p), -(-Wo // p)
    padb = (nhy - 1) * q + T - H + lo
    padr = (nhx - 1) * q + T - W + lo
    xt = torch.from_numpy(x)[:, None]
    if padb < 0:
        xt = xt[..., : H + padb, :]
        padb = 0
    if padr < 0:
        xt = xt[..., :, : W + padr]
        padr = 0
    tmode = {"zero": "constant", "replicate": "replicate", "reflect": "reflect"}[pad]
    y = F.pixel_shuffle(F.conv2d(F.pad(xt, (-lo, padr, -lo, padb), mode=tmode), w, stride=q), p)[:, 0, :Ho, :Wo]
    (y * torch.from_numpy(g)).sum().backward()
    gw = w.grad.numpy()[:, 0]  # (p*p, T, T)
    nt = {"nearest": 1, "bilinear": 2, "bicubic": 4}[mode]
    out = np.empty((p, p, nt, nt))
    for jy, jx in itertools.product(range(p), range(p)):
        fy = oracle.phase_taps(mode, p, q, jy)[0] - lo
        fx = oracle.phase_taps(mode, p, q, jx)[0] - lo
        out[jy, jx] = gw[jy * p + jx, fy:fy + nt, fx:fx + nt]
    return out


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("pad", PADS)
def test_weight_grad_equals_torch_autograd_of_the_layer(mode, pad):
    for n, ((p, q), ext) in enumerate(itertools.product([(3, 2), (2, 3), (5, 3), (3, 5), (4, 1)], (False, True))):
        H, W = 13, 17
        x = rnd(70 + n, (2, H, W))
        Ho, Wo = oracle.output_shape(H, W, p, q, ext)
        g = rnd(90 + n, (2, Ho, Wo))
        ours, ab = oracle.weight_grad(x, g, p, q, mode, pad, floor_extent=ext)
        ref = torch_layer_wgrad(x, g, p, q, mode, pad, ext)
        np.testing.assert_allclose(ours, ref, rtol=0, atol=1e-12, err_msg=f"{p}/{q} {mode} {pad} {ext}")
        assert (ab >= np.abs(ours) - 1e-12).all()


def test_weight_grad_closed_forms():
    # nearest p/1: output (p*i + jy, p*k + jx) copies x[i, k]
    for p in (2, 3):
        x = rnd(11, (3, 5, 6))
        g = rnd(12, (3, 5 * p, 6 * p))
        ours, _ = oracle.weight_grad(x, g, p, 1, "nearest", "zero")
        want = np.einsum("nikab,nik->ab", g.reshape(3, 5, p, 6, p).transpose(0, 1, 3, 2, 4), x)
        np.testing.assert_allclose(ours[:, :, 0, 0], want, rtol=0, atol=1e-12)
    # identity 1/1, bilinear taps {0, +1} (second weight 0), replicate: sum g[m] x~[m + (a, b)]
    x = rnd(13, (2, 7, 8))
    g = rnd(14, (2, 7, 8))
    xp = np.pad(x, ((0, 0), (0, 1), (0, 1)), mode="edge")
    ours, _ = oracle.weight_grad(x, g, 1, 1, "bilinear", "replicate")
    for a, b in itertools.product(range(2), range(2)):
        assert abs(ours[0, 0, a, b] - (g * xp[:, a:a + 7, b:b + 8]).sum()) < 1e-12


def test_weight_grad_1d_and_linearity():
    x = rnd(15, (2, 3, 40))
    for mode, (p, q) in itertools.product(MODES, [(3, 2), (2, 3), (5, 3)]):
        Wo = oracle.output_extent(40, p, q, True)
        g1, g2 = rnd(16, (2, 3, Wo)), rnd(17, (2, 3, Wo))
        a1, _ = oracle.weight_grad(x, g1, p, q, mode, "reflect", floor_extent=True, is1d=True)
        a2, _ = oracle.weight_grad(x, g2, p, q, mode, "reflect", floor_extent=True, is1d=True)
        a12, _ = oracle.weight_grad(x, 2 * g1 - g2, p, q, mode, "reflect", floor_extent=True, is1d=True)
        np.testing.assert_allclose(a12, 2 * a1 - a2, rtol=0, atol=1e-11)
        # 1D = the 2D formula on rows (torch conv1d through conv2d with a 1-row kernel)
        ref = np.zeros_like(a1)
        kers = [oracle.phase_taps(mode, p, q, j) for j in range(p)]
        for j, (first, w) in enumerate(kers):
            for t in range(len(w)):
                for m in range(j, Wo, p):
                    v = (m // p) * q + first + t
                    v = -v if v < 0 else (2 * 39 - v if v > 39 else v)
                    ref[0, j, 0, t] += (g1[..., m] * x[..., v]).sum()
        np.testing.assert_allclose(a1, ref, rtol=0, atol=1e-11)


def torch_layer_wgrad_2d(x, g, p, q, mode, pad, ext):
    """torch float64 autograd through the anisotropic layer: F.pad -> F.conv2d
    (stride (qy, qx), a (py*px, 1, Ty, Tx) weight) -> pixelshuffle by (py, px)
    as reshape/permute -> crop; the weight's .grad read at each phase's taps."""
    import torch
    import torch.nn.functional as F
    (py, px), (qy, qx) = p, q
    N, H, W = x.shape
    Ho, Wo = oracle.output_extent(H, py, qy, ext), oracle.output_extent(W, px, qx, ext)
    def win(pp, qq):
        firsts = [oracle.phase_taps(mode, pp, qq, j)[0] for j in range(pp)]
        nt = len(oracle.phase_taps(mode, pp, qq, 0)[1])
        lo, hi = min(firsts), max(firsts) + nt - 1
        return firsts, lo, hi - lo + 1, nt
    fy, loy, Ty, nt = win(py, qy)
    fx, lox, Tx, _ = win(px, qx)
    k = np.zeros((py * px, 1, Ty, Tx))
    for jy in range(py):
        for jx in range(px):
            wy = oracle.phase_taps(mode, py, qy, jy)[1]
            wx = oracle.phase_taps(mode, px, qx, jx)[1]
            k[jy * px + jx, 0, fy[jy] - loy:fy[jy] - loy + nt, fx[jx] - lox:fx[jx] - lox + nt] = np.outer(wy, wx)
    w = torch.from_numpy(k).requires_grad_(True)
    nhy, nhx = -(-Ho // py), -(-Wo // px)
    padb, padr = (nhy - 1) * qy + Ty - H + loy, (nhx - 1) * qx + Tx - W + lox
    xt = torch.from_numpy(x)[:, None]
    if padb < 0:
        xt, padb = xt[..., : H + padb, :], 0
    if padr < 0:
        xt, padr = xt[..., :, : W + padr], 0
    tmode = {"zero": "constant", "replicate": "replicate", "reflect": "reflect"}[pad]
    h = F.conv2d(F.pad(xt, (-lox, padr, -loy, padb), mode=tmode), w, stride=(qy, qx))  # (N, py*px, nhy, nhx)
    y = h.reshape(N, py, px, nhy, nhx).permute(0, 3, 1, 4, 2).reshape(N, nhy * py, nhx * px)[:, :Ho, :Wo]
    (y * torch.from_numpy(g)).sum().backward()
    gw = w.grad.numpy()[:, 0]
    out = np.empty((py, px, nt, nt))
    for jy in range(py):
        for jx in range(px):
            out[jy, jx] = gw[jy * px + jx, fy[jy] - loy:fy[jy] - loy + nt, fx[jx] - lox:fx[jx] - lox + nt]
    return out


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("pad", PADS)
def test_weight_grad_2d_anisotropic_equals_torch_autograd(mode, pad):
    for n, (p, q, ext) in enumerate([((5, 2), (3, 7), False), ((3, 4), (2, 3), True), ((2, 7), (5, 4), True),
                                      ((4, 1), (1, 3), False)]):
        H, W = 17, 23
        x = rnd(200 + n, (2, H, W))
        Ho, Wo = oracle.output_extent(H, p[0], q[0], ext), oracle.output_extent(W, p[1], q[1], ext)
        g = rnd(220 + n, (2, Ho, Wo))
        try:
            ours, ab = oracle.weight_grad_2d(x, g, p, q, mode, pad, floor_extent=ext)
        except oracle.OracleError as e:
            assert pad == "reflect" and e.code == -2
            continue
        ref = torch_layer_wgrad_2d(x, g, p, q, mode, pad, ext)
        np.testing.assert_allclose(ours, ref, rtol=0, atol=1e-12, err_msg=f"{p}/{q} {mode} {pad}")
