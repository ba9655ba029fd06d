"""Pins of the oracle's ND / per-dimension-factor evaluators (§4.2).

"To scale an ND input signal by scaling factors r_1/s_1, ..., r_n/s_n for the
different dimensions": pad -> conv with prod r_i output channels and stride
[s_1..s_n] -> ND pixelshuffle (§4.1).  As for the 2D oracle,
nothing here compares the oracle with a retyped copy of itself: the ND staged
evaluator is checked against the independent direct evaluator, against the
separately pinned 1D code path applied once per axis (separability), against
exact index gathers, scipy.ndimage.map_coordinates (order 1), torch float64
F.pad -> F.conv3d -> a 3D pixel shuffle, and exact rational brute force.  A
factor applied to the wrong axis, a transposed channel order or a dropped tap
fails at least one of them.
"""
import itertools
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

MODES = ["nearest", "bilinear", "bicubic"]
PADS = ["zero", "replicate", "reflect"]
FACTORS = [(1, 1), (3, 2), (2, 3), (5, 3), (3, 5), (4, 7), (7, 4), (2, 1), (1, 3)]


def rng_input(seed, shape):
    return synth.uniform_f32(seed, int(np.prod(shape))).reshape(shape).astype(np.float64)


def _1d_along(x, axis, p, q, mode, pad, floor_extent):
    """The oracle's 1D path (§3.1, pinned in test_oracle_pins) along one axis."""
    xm = np.moveaxis(x, axis, -1)
    y = oracle.staged(np.ascontiguousarray(xm), p, q, mode, pad, floor_extent=floor_extent, is1d=True)
    return np.moveaxis(y, -1, axis)


def test_nd_staged_equals_direct_sweep():
    rs = np.random.RandomState(21)
    n = 0
    for R in (1, 2, 3):
        for mode, pad in itertools.product(MODES, PADS):
            for _ in range(3):
                fac = [FACTORS[i] for i in rs.randint(0, len(FACTORS), size=R)]
                p, q = [f[0] for f in fac], [f[1] for f in fac]
                dims = tuple(int(v) for v in rs.randint(2, 9 if R == 3 else 17, size=R))
                x = rng_input(300 + n, (2,) + dims)
                n += 1
                for ext in (False, True):
                    try:
                        a = oracle.staged_nd(x, p, q, mode, pad, floor_extent=ext)
                    except oracle.OracleError as e:
                        assert e.code in (-2, -3)
                        with pytest.raises(oracle.OracleError):
                            oracle.direct_nd(x, p, q, mode, pad, floor_extent=ext)
                        continue
                    b = oracle.direct_nd(x, p, q, mode, pad, floor_extent=ext)
                    assert a.shape == b.shape == (2,) + oracle.output_dims_nd(dims, p, q, ext)
                    np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)
    assert n == 3 * 9 * 3


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("pad", ["zero", "replicate", "reflect"])
def test_nd_is_separable_into_1d_passes(mode, pad):
    """§4.2 kernels are outer products, so the ND layer equals the 1D layer
    (§3.1) applied along each axis with that axis' own factor."""
    x = rng_input(31, (2, 7, 9, 11))
    for p, q in [((3, 2, 5), (2, 3, 3)), ((1, 4, 3), (1, 7, 5)), ((2, 1, 1), (1, 1, 2))]:
        for ext in (False, True):
            nd = oracle.staged_nd(x, p, q, mode, pad, floor_extent=ext)
            y = x
            for axis, (pp, qq) in zip((-1, -2, -3), zip(p[::-1], q[::-1])):
                y = _1d_along(y, axis, pp, qq, mode, pad, ext)
            np.testing.assert_allclose(nd, y, rtol=0, atol=1e-13)
    # anisotropic 2D likewise
    x2 = rng_input(32, (3, 13, 10))
    nd = oracle.staged_nd(x2, (5, 2), (3, 7), mode, pad)
    y = _1d_along(_1d_along(x2, -1, 2, 7, mode, pad, False), -2, 5, 3, mode, pad, False)
    np.testing.assert_allclose(nd, y, rtol=0, atol=1e-13)


def test_rank1_and_isotropic_rank2_match_the_1d_and_2d_paths():
    x = rng_input(33, (4, 6, 29))
    for mode, pad in itertools.product(MODES, PADS):
        for (p, q) in [(3, 2), (5, 3), (3, 5)]:
            np.testing.assert_allclose(oracle.staged_nd(x, [p], [q], mode, pad),
                                       oracle.staged(x, p, q, mode, pad, is1d=True), rtol=0, atol=1e-13)
            np.testing.assert_allclose(oracle.staged_nd(x, [p, p], [q, q], mode, pad),
                                       oracle.staged(x, p, q, mode, pad), rtol=0, atol=1e-13)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("pad", PADS)
def test_nd_identity_is_exact(mode, pad):
    x = rng_input(34, (2, 4, 5, 6))
    for ext in (False, True):
        assert np.array_equal(oracle.staged_nd(x, (1, 1, 1), (1, 1, 1), mode, pad, floor_extent=ext), x)
        assert np.array_equal(oracle.staged_nd(x, (2, 3, 4), (2, 3, 4), mode, pad, floor_extent=ext), x)


@pytest.mark.parametrize("pad", PADS)
def test_nd_nearest_is_an_index_gather(pad):
    """Nearest (§5.2.1, reading Z2) in 3D takes x[floor(m_z q_z/p_z), floor(m_y q_y/p_y), floor(m_x q_x/p_x)]."""
    x = rng_input(35, (2, 6, 7, 9))
    for p, q in [((3, 2, 5), (2, 3, 3)), ((2, 1, 3), (1, 2, 4)), ((4, 3, 1), (7, 5, 1))]:
        for ext in (False, True):
            y = oracle.staged_nd(x, p, q, "nearest", pad, floor_extent=ext)
            idx = [np.array([(m * qq) // pp for m in range(no)]) for no, pp, qq in zip(y.shape[1:], p, q)]
            # indices past the end exist only in the paper extent: they read padding
            ok = [i < n for i, n in zip(idx, x.shape[1:])]
            ref = x[:, idx[0][ok[0]]][:, :, idx[1][ok[1]]][:, :, :, idx[2][ok[2]]]
            np.testing.assert_array_equal(y[:, ok[0]][:, :, ok[1]][:, :, :, ok[2]], ref)


@pytest.mark.parametrize("pad", PADS)
def test_trilinear_equals_scipy_map_coordinates(pad):
    from scipy import ndimage
    x = rng_input(36, (6, 7, 9))
    for p, q in [((3, 2, 5), (2, 3, 3)), ((4, 5, 7), (7, 3, 5))]:
        ours = oracle.staged_nd(x, p, q, "bilinear", pad, floor_extent=True)
        g = np.mgrid[0:ours.shape[0], 0:ours.shape[1], 0:ours.shape[2]].astype(np.float64)
        coords = [g[d] * q[d] / p[d] for d in range(3)]
        smode = {"zero": "grid-constant", "replicate": "nearest", "reflect": "mirror"}[pad]
        ref = ndimage.map_coordinates(x, coords, order=1, mode=smode, cval=0.0)
        np.testing.assert_allclose(ours, ref, rtol=0, atol=1e-12)


def _torch_layer_3d(x, p, q, mode, pad, floor_extent):
    """The paper's ND layer with torch float64 library ops: F.pad ->
    F.conv3d (p0*p1*p2 channels, stride q) -> 3D pixel shuffle -> crop.  The
    3D kernels are outer products (einsum) of the 1D phase kernels."""
    import torch
    import torch.nn.functional as F
    dims = x.shape
    odims = oracle.output_dims_nd(dims, p, q, floor_extent)
    k1, lo, T = [], [], []
    for pp, qq in zip(p, q):
        taps = [oracle.phase_taps(mode, pp, qq, j) for j in range(pp)]
        l = min(f for f, _ in taps)
        h = max(f + len(w) - 1 for f, w in taps)
        ks = np.zeros((pp, h - l + 1))
        for j, (f, w) in enumerate(taps):
            ks[j, f - l: f - l + len(w)] = w
        k1.append(ks)
        lo.append(l)
        T.append(h - l + 1)
    wt = np.einsum("ai,bj,ck->abcijk", *k1).reshape(p[0] * p[1] * p[2], 1, T[0], T[1], T[2])
    nh = [-(-o // pp) for o, pp in zip(odims, p)]
    before = [-l for l in lo]
    after = [(n - 1) * qq + t - d - b for n, qq, t, d, b in zip(nh, q, T, dims, before)]
    xt = torch.from_numpy(x)[None, None]
    sl = [slice(None)] * 2 + [slice(0, d + a) if a < 0 else slice(None) for d, a in zip(dims, after)]
    xt = xt[tuple(sl)]
    after = [max(a, 0) for a in after]
    tmode = {"zero": "constant", "replicate": "replicate", "reflect": "reflect"}[pad]
    xp = F.pad(xt, (before[2], after[2], before[1], after[1], before[0], after[0]), mode=tmode)
    hid = F.conv3d(xp, torch.from_numpy(wt), stride=tuple(q))[0]            # (p0 p1 p2, n0, n1, n2)
    h = hid.reshape(p[0], p[1], p[2], nh[0], nh[1], nh[2]).permute(3, 0, 4, 1, 5, 2)
    out = h.reshape(nh[0] * p[0], nh[1] * p[1], nh[2] * p[2])
    return out[: odims[0], : odims[1], : odims[2]].numpy()


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("pad", PADS)
def test_nd_equals_torch_pad_conv3d_shuffle(mode, pad):
    x = rng_input(37, (7, 8, 10))
    for p, q in [((3, 2, 5), (2, 3, 3)), ((2, 5, 1), (3, 4, 1))]:
        for ext in (False, True):
            try:
                ours = oracle.staged_nd(x, p, q, mode, pad, floor_extent=ext)
            except oracle.OracleError as e:
                assert pad == "reflect" and e.code == -2
                continue
            np.testing.assert_allclose(ours, _torch_layer_3d(x, p, q, mode, pad, ext), rtol=0, atol=1e-12)


def _keys(d):
    d = abs(d)
    a = Fraction(-1, 2)
    if d <= 1:
        return (a + 2) * d ** 3 - (a + 3) * d ** 2 + 1
    if d < 2:
        return a * d ** 3 - 5 * a * d ** 2 + 8 * a * d - 4 * a
    return Fraction(0)


def _exact_nd(x, p, q, mode, pad, m):
    dims = x.shape

    def rm(t, n):
        if 0 <= t < n:
            return t
        if pad == "zero":
            return None
        if pad == "replicate":
            return 0 if t < 0 else n - 1
        return -t if t < 0 else 2 * (n - 1) - t

    taps = {"nearest": [0], "bilinear": [0, 1], "bicubic": [-1, 0, 1, 2]}[mode]
    u = [Fraction(mm * qq, pp) for mm, pp, qq in zip(m, p, q)]
    b = [int(v) for v in u]
    acc = Fraction(0)
    for t in itertools.product(taps, repeat=len(dims)):
        w = Fraction(1)
        for d in range(len(dims)):
            if mode == "bilinear":
                w *= 1 - abs(u[d] - (b[d] + t[d]))
            elif mode == "bicubic":
                w *= _keys(u[d] - (b[d] + t[d]))
        src = [rm(b[d] + t[d], dims[d]) for d in range(len(dims))]
        if any(s is None for s in src):
            continue
        acc += w * Fraction(int(x[tuple(src)]))
    return acc


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("pad", PADS)
def test_nd_exact_rational_brute_force(mode, pad):
    rs = np.random.RandomState(38)
    for shape, p, q in [((5, 6), (5, 2), (3, 7)), ((4, 3, 5), (3, 2, 5), (2, 3, 3))]:
        x = rs.randint(-9, 10, size=shape).astype(np.float64)
        try:
            y = oracle.staged_nd(x, p, q, mode, pad, floor_extent=True)
        except oracle.OracleError as e:
            assert pad == "reflect" and e.code == -2
            continue
        for m in itertools.product(*[range(n) for n in y.shape]):
            e = _exact_nd(x, p, q, mode, pad, m)
            assert abs(y[m] - float(e)) <= 1e-12 * max(1.0, abs(float(e)))
