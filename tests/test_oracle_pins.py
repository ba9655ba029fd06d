"""Pins of the CPU oracle (oracle/) against what the paper and mathematics fix.

None of these compares the oracle with itself or with a retyped copy of its
formula alone: values printed in the paper (tests/golden/paper_values.json,
each cited), closed-form properties (identity, pixel repetition, constants,
ramps, quadratics, linearity, separability), library routines that reduce to
special cases (numpy repeat, scipy.ndimage.map_coordinates order 1, torch
float64 pad -> conv2d -> pixel_shuffle, torch nearest interpolate), and exact
rational brute force on tiny inputs.  A dropped term, wrong sign, wrong index
or transposed operand in the oracle fails at least one of them.
"""
import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
MODES = ["nearest", "bilinear", "bicubic"]
PADS = ["zero", "replicate", "reflect"]


def rng_input(seed, shape):
    return synth.uniform_f32(seed, int(np.prod(shape))).reshape(shape).astype(np.float64)


def frac_of(j, p, q):
    """phase j's fraction as a pair, from the oracle's taps (bilinear weight f)."""
    _, w = oracle.phase_taps("bilinear", p, q, j)
    return w[1]


# ----------------------------------------------------------------- §5.2 weights
def test_bilinear_kernels_match_paper_printout():
    g = GOLD["bilinear_3_2"]
    p, q = 3, 2
    # locate the phases whose fractions are 1/3 and 2/3 (reading Z1)
    fr = {j: frac_of(j, p, q) for j in range(p)}
    j13 = [j for j in fr if abs(fr[j] - 1 / 3) < 1e-12][0]
    j23 = [j for j in fr if abs(fr[j] - 2 / 3) < 1e-12][0]
    for (jy, jx), printed in [((j13, j13), g["W11"]), ((j13, j23), g["W13"])]:
        T, lo, K = oracle.kernel2d("bilinear", p, q, jy, jx)
        nz = K[np.ix_(np.any(K != 0, axis=1), np.any(K != 0, axis=0))]
        assert nz.shape == (2, 2)
        np.testing.assert_array_equal(np.round(nz, g["decimals"]), np.array(printed))
    # exact values behind the 2-decimal printout: outer products of (2/3, 1/3)
    T, lo, K = oracle.kernel2d("bilinear", p, q, j13, j13)
    nz = K[np.ix_(np.any(K != 0, axis=1), np.any(K != 0, axis=0))]
    np.testing.assert_allclose(nz, [[4 / 9, 2 / 9], [2 / 9, 1 / 9]], rtol=0, atol=1e-15)


def test_nearest_kernels_match_paper_printout():
    g = GOLD["nearest_3_2"]
    p, q = 3, 2
    kernels = [oracle.kernel2d("nearest", p, q, jy, jx) for jy in range(p) for jx in range(p)]
    assert len(kernels) == g["count"]
    for T, lo, K in kernels:  # every kernel is one-hot
        assert np.count_nonzero(K) == 1 and K.sum() == 1.0
    # phase (0,0): one-hot at the window origin, [[1,0],[0,0]]
    T, lo, K = oracle.kernel2d("nearest", p, q, 0, 0)
    np.testing.assert_array_equal(K[:2, :2], g["W11"])
    # a phase whose x-tap moved by one pixel gives [[0,1],[0,0]]
    found = False
    for jx in range(p):
        T, lo, K = oracle.kernel2d("nearest", p, q, 0, jx)
        if np.array_equal(K[:2, :2], np.array(g["W13"])):
            found = True
    assert found


def test_bicubic_weight_matches_paper_formula():
    g = GOLD["bicubic_W"]
    c3, c2, c1, c0 = g["branch1_coeffs_d3_d2_d1_d0"]
    for d in np.linspace(0.0, 1.0, 17):
        assert oracle.cubic_weight(d) == pytest.approx(c3 * d ** 3 + c2 * d ** 2 + c1 * d + c0, abs=1e-15)
        assert oracle.cubic_weight(-d) == oracle.cubic_weight(d)  # W depends on |Delta|
    b3, b2, b1 = g["branch2_coeffs_d3_d2_d1"]
    a = -0.5  # reading Z7
    for d in np.linspace(1.0625, 1.9375, 15):
        assert oracle.cubic_weight(d) == pytest.approx(b3 * d ** 3 + b2 * d ** 2 + b1 * d - 4 * a, abs=1e-14)
    assert oracle.cubic_weight(2.0) == 0.0 and oracle.cubic_weight(3.7) == 0.0
    # continuity at the branch points and the interpolation property W(0)=1, W(1)=W(2)=0
    assert oracle.cubic_weight(1.0) == 0.0 and oracle.cubic_weight(0.0) == 1.0
    assert oracle.cubic_weight(1 + 1e-12) == pytest.approx(0.0, abs=1e-11)
    assert oracle.cubic_weight(2 - 1e-12) == pytest.approx(0.0, abs=1e-11)


def test_spec_weight_examples():
    for c in GOLD["spec_cubic_weight"]["cases"]:
        assert oracle.cubic_weight(c["delta"]) == c["w"]
    for c in GOLD["spec_phase_fraction"]["cases"]:
        assert frac_of(c["j"], c["p"], c["q"]) == pytest.approx(c["frac"][0] / c["frac"][1], abs=1e-15)
    # weights_1d at a fraction: find p, q, j giving that fraction
    for c in GOLD["spec_weights_1d"]["cases"]:
        num, den = c["frac"]
        p, q, j = den, num, 1  # j*q mod p / p = num/den
        first, w = oracle.phase_taps(c["mode"], p, q, j)
        np.testing.assert_allclose(w, c["w"], atol=1e-15)


@pytest.mark.parametrize("mode", ["bilinear", "bicubic"])
@pytest.mark.parametrize("p,q", [(3, 2), (5, 3), (7, 5), (4, 7), (3, 5), (27, 11), (2, 11)])
def test_partition_of_unity_and_symmetry(mode, p, q):
    for j in range(p):
        first, w = oracle.phase_taps(mode, p, q, j)
        assert abs(w.sum() - 1.0) < 1e-14
        f = frac_of(j, p, q)
        # weights at f reversed equal the weights at 1-f; find phase with 1-f
        for j2 in range(p):
            if f > 0 and abs(frac_of(j2, p, q) - (1 - f)) < 1e-14:
                _, w2 = oracle.phase_taps(mode, p, q, j2)
                np.testing.assert_allclose(w[::-1], w2, atol=1e-15)


def test_bicubic_half_fraction_closed_form():
    first, w = oracle.phase_taps("bicubic", 2, 1, 1)  # f = 1/2
    assert first == -1
    np.testing.assert_array_equal(w, [-1 / 16, 9 / 16, 9 / 16, -1 / 16])


# ----------------------------------------------------------------- §3 primitives
def test_pad_examples():
    for c in GOLD["spec_pad"]["cases"]:
        np.testing.assert_array_equal(oracle.pad1d(c["x"], c["left"], c["right"], c["pad"]), c["out"])


def test_reflect_infeasible_raises():
    with pytest.raises(oracle.OracleError):
        oracle.pad1d([1.0, 2.0], 2, 0, "reflect")


def test_strided_conv_examples():
    for c in GOLD["spec_strided_conv"]["cases"]:
        np.testing.assert_array_equal(oracle.strided_conv1d(c["x"], c["kernels"], c["stride"]), c["out"])


def test_pixelshuffle_examples_and_figures():
    for c in GOLD["spec_pixelshuffle"]["cases"]:
        h = np.array(c["h"], dtype=np.float64)[:, 0, :]  # (4, 1, 1) -> (4, 1, 1)
        h = np.array(c["h"], dtype=np.float64).reshape(4, 1, 1)
        np.testing.assert_array_equal(oracle.pixelshuffle2d(h, *c["r"]), c["out"])
    g = GOLD["pixelshuffle_fig3"]
    h = np.array([[7.0], [8.0], [9.0]])
    out = oracle.pixelshuffle1d(h)
    assert list(out.shape) == g["out_shape"] and list(out) == [7.0, 8.0, 9.0]
    g = GOLD["pixelshuffle_fig4"]
    h = np.arange(np.prod(g["in_shape"]), dtype=np.float64).reshape(g["in_shape"])
    out = oracle.pixelshuffle2d(h, 3, 3)
    assert list(out.shape) == g["out_shape"]
    # a permutation that agrees with torch's pixel_shuffle (reading Z10)
    import torch
    ref = torch.nn.functional.pixel_shuffle(torch.from_numpy(h)[None], 3)[0, 0].numpy()
    np.testing.assert_array_equal(out, ref)


def test_pixelshuffle_roundtrip_with_torch_unshuffle():
    import torch
    for (r, n1, n2) in [(2, 3, 4), (3, 1, 5), (4, 2, 2)]:
        x = torch.arange(r * n1 * r * n2, dtype=torch.float64).reshape(1, 1, r * n1, r * n2)
        h = torch.nn.functional.pixel_unshuffle(x, r)[0].numpy()
        np.testing.assert_array_equal(oracle.pixelshuffle2d(h, r, r), x[0, 0].numpy())


# ----------------------------------------------------------------- shapes
def test_paper_shape_example():
    g = GOLD["shape_example"]
    H, W = g["in"]
    x = rng_input(1, (H, W))
    for mode in MODES:
        out = oracle.staged(x, g["p"], g["q"], mode, "replicate", floor_extent=False)
        assert list(out.shape) == g["out_paper_extent"]


def test_spec_output_shapes():
    for c in GOLD["spec_output_shape"]["cases"]:
        assert oracle.output_extent(c["n"], c["p"], c["q"], False) == c["out"]
    for c in GOLD["baseline_shapes"]["cases"]:
        assert list(oracle.output_shape(c["H"], c["W"], c["p"], c["q"], c["floor"])) == c["out"]


def test_spec_scale_examples():
    for c in GOLD["spec_scale"]["cases"]:
        x = np.array([c["x"]], dtype=np.float64)
        for fn in (oracle.staged, oracle.direct):
            y = fn(x, c["p"], c["q"], c["mode"], c["pad"], floor_extent=False, is1d=True)
            np.testing.assert_allclose(y[0], c["out"], atol=1e-14)


# ----------------------------------------------------------------- closed forms
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("pad", PADS)
@pytest.mark.parametrize("pq", [(1, 1), (3, 3), (7, 7)])
def test_identity_is_exact(mode, pad, pq):
    x = rng_input(2, (2, 9, 13))
    for ext in (False, True):
        for is1d in (False, True):
            y = oracle.staged(x, *pq, mode, pad, floor_extent=ext, is1d=is1d)
            np.testing.assert_array_equal(y, x)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 7])
def test_integer_nearest_is_pixel_repetition(p):
    x = rng_input(3, (2, 5, 6))
    rep = np.repeat(np.repeat(x, p, axis=-2), p, axis=-1)
    for ext in (False, True):
        np.testing.assert_array_equal(oracle.staged(x, p, 1, "nearest", "zero", floor_extent=ext), rep)
        np.testing.assert_array_equal(oracle.direct(x, p, 1, "nearest", "zero", floor_extent=ext), rep)


@pytest.mark.parametrize("p,q", [(3, 2), (2, 3), (5, 3), (3, 5), (7, 5), (4, 7), (27, 11), (2, 11)])
def test_nearest_matches_torch_interpolate_indices(p, q):
    import torch
    H, W = 22, 33
    x = torch.arange(H * W, dtype=torch.float64).reshape(1, 1, H, W)
    ref = torch.nn.functional.interpolate(x, scale_factor=p / q, mode="nearest")
    ours = oracle.staged(x.numpy()[0], p, q, "nearest", "replicate", floor_extent=True)
    assert ours.shape[-2:] == tuple(ref.shape[-2:])
    np.testing.assert_array_equal(ours, ref[0].numpy())


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("pad", ["replicate", "reflect"])
@pytest.mark.parametrize("p,q", [(3, 2), (5, 3), (3, 5), (4, 7)])
def test_constants_are_preserved(mode, pad, p, q):
    x = np.full((11, 14), 0.3712)
    y = oracle.staged(x, p, q, mode, pad)
    np.testing.assert_allclose(y, 0.3712, rtol=0, atol=1e-15)


def _interior_mask(Ho, Wo, H, W, p, q, lo, hi):
    """Outputs whose own taps all fall inside the image."""
    my = np.arange(Ho)
    mx = np.arange(Wo)
    by = (my * q) // p
    bx = (mx * q) // p
    oky = (by + lo >= 0) & (by + hi <= H - 1)
    okx = (bx + lo >= 0) & (bx + hi <= W - 1)
    return oky[:, None] & okx[None, :]


@pytest.mark.parametrize("p,q", [(3, 2), (5, 3), (7, 5), (4, 7), (3, 5), (2, 11), (27, 11)])
def test_bilinear_reproduces_ramps(p, q):
    H, W = 23, 29
    i, j = np.mgrid[0:H, 0:W].astype(np.float64)
    x = 0.25 + 1.5 * i - 0.75 * j
    for pad in PADS:
        y = oracle.staged(x, p, q, "bilinear", pad)
        Ho, Wo = y.shape
        my, mx = np.mgrid[0:Ho, 0:Wo].astype(np.float64)
        expect = 0.25 + 1.5 * (my * q / p) - 0.75 * (mx * q / p)
        m = _interior_mask(Ho, Wo, H, W, p, q, 0, 1)
        assert m.sum() > 0
        np.testing.assert_allclose(y[m], expect[m], rtol=0, atol=1e-11)


@pytest.mark.parametrize("p,q", [(3, 2), (5, 3), (7, 5), (3, 5), (27, 11)])
def test_bicubic_reproduces_quadratics(p, q):
    # Keys' kernel with a = -1/2 reproduces polynomials up to degree 2 per dimension
    H, W = 21, 26
    i, j = np.mgrid[0:H, 0:W].astype(np.float64)
    f = lambda a, b: 1 + 0.2 * a - 0.5 * b + 0.03 * a * a - 0.02 * b * b + 0.01 * a * b
    x = f(i, j)
    y = oracle.staged(x, p, q, "bicubic", "replicate")
    Ho, Wo = y.shape
    my, mx = np.mgrid[0:Ho, 0:Wo].astype(np.float64)
    m = _interior_mask(Ho, Wo, H, W, p, q, -1, 2)
    assert m.sum() > 0
    np.testing.assert_allclose(y[m], f(my * q / p, mx * q / p)[m], rtol=0, atol=1e-11)
    # ... but not cubics (a = -1/2 is third-order accurate, not exact): a sanity
    # check that the test above can fail.
    xc = i ** 3
    yc = oracle.staged(xc, p, q, "bicubic", "replicate")
    assert np.abs(yc[m] - ((my * q / p) ** 3)[m]).max() > 1e-3


def test_linearity():
    x = rng_input(4, (3, 17, 19))
    z = rng_input(5, (3, 17, 19))
    for mode, pad in itertools.product(MODES, PADS):
        a = oracle.staged(2.5 * x - 0.75 * z, 5, 3, mode, pad)
        b = 2.5 * oracle.staged(x, 5, 3, mode, pad) - 0.75 * oracle.staged(z, 5, 3, mode, pad)
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("pad", PADS)
def test_separability_2d_equals_1d_twice(mode, pad):
    x = rng_input(6, (2, 15, 18))
    for (p, q) in [(3, 2), (5, 3), (3, 5)]:
        two = oracle.staged(x, p, q, mode, pad)
        rows = oracle.staged(x, p, q, mode, pad, is1d=True)                   # along W
        cols = oracle.staged(np.ascontiguousarray(np.swapaxes(rows, -1, -2)), p, q, mode, pad, is1d=True)
        np.testing.assert_allclose(two, np.swapaxes(cols, -1, -2), rtol=0, atol=1e-13)


# ----------------------------------------------------------------- independent implementations
def test_staged_equals_direct_sweep():
    rs = np.random.RandomState(7)
    facs = [(1, 1), (3, 2), (2, 3), (3, 4), (5, 3), (7, 5), (4, 7), (3, 5), (2, 11), (27, 11), (2, 1), (3, 1), (1, 4)]
    n = 0
    for (p, q) in facs:
        for mode, pad in itertools.product(MODES, PADS):
            H, W = rs.randint(2, 25, size=2)
            x = rng_input(100 + n, (2, H, W))
            n += 1
            for ext, is1d in itertools.product((False, True), (False, True)):
                try:
                    a = oracle.staged(x, p, q, mode, pad, floor_extent=ext, is1d=is1d)
                except oracle.OracleError as e:
                    # only infeasible reflect or an empty floor extent may refuse
                    assert e.code in (-2, -3)
                    with pytest.raises(oracle.OracleError):
                        oracle.direct(x, p, q, mode, pad, floor_extent=ext, is1d=is1d)
                    continue
                b = oracle.direct(x, p, q, mode, pad, floor_extent=ext, is1d=is1d)
                np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)
    assert n == len(facs) * 9


def _torch_layer(x, p, q, mode, pad, floor_extent):
    """The paper's single layer with torch float64 library ops: F.pad ->
    F.conv2d (p*p output channels, stride q) -> F.pixel_shuffle -> crop."""
    import torch
    import torch.nn.functional as F
    H, W = x.shape
    Ho, Wo = oracle.output_shape(H, W, p, q, floor_extent)
    kers = [oracle.kernel2d(mode, p, q, jy, jx) for jy in range(p) for jx in range(p)]
    T, lo = kers[0][0], kers[0][1]
    wt = torch.from_numpy(np.stack([k[2] for k in kers]))[:, None]
    nhy, nhx = -(-Ho // p), -(-Wo // p)
    padt = -lo
    padb = (nhy - 1) * q + T - H - padt
    padl = -lo
    padr = (nhx - 1) * q + T - W - padl
    xt = torch.from_numpy(x)[None, None]
    tmode = {"zero": "constant", "replicate": "replicate", "reflect": "reflect"}[pad]
    # crop first if the window needs less than the image (negative pads)
    if padb < 0:
        xt = xt[..., : H + padb, :]
        padb = 0
    if padr < 0:
        xt = xt[..., :, : W + padr]
        padr = 0
    xp = F.pad(xt, (padl, padr, padt, padb), mode=tmode)
    hid = F.conv2d(xp, wt, stride=q)
    return F.pixel_shuffle(hid, p)[0, 0, :Ho, :Wo].numpy()


@pytest.mark.parametrize("p,q", [(3, 2), (2, 3), (5, 3), (7, 5), (4, 7), (3, 5), (27, 11)])
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("pad", PADS)
def test_staged_equals_torch_pad_conv_shuffle(p, q, mode, pad):
    x = rng_input(8, (19, 23))
    for ext in (False, True):
        ours = oracle.staged(x, p, q, mode, pad, floor_extent=ext)
        ref = _torch_layer(x, p, q, mode, pad, ext)
        np.testing.assert_allclose(ours, ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("p,q", [(3, 2), (5, 3), (7, 5), (4, 7), (3, 5)])
@pytest.mark.parametrize("pad", PADS)
def test_bilinear_equals_scipy_map_coordinates(p, q, pad):
    from scipy import ndimage
    x = rng_input(9, (17, 21))
    ours = oracle.staged(x, p, q, "bilinear", pad, floor_extent=True)
    Ho, Wo = ours.shape
    my, mx = np.mgrid[0:Ho, 0:Wo].astype(np.float64)
    smode = {"zero": "grid-constant", "replicate": "nearest", "reflect": "mirror"}[pad]
    ref = ndimage.map_coordinates(x, [my * q / p, mx * q / p], order=1, mode=smode, cval=0.0)
    np.testing.assert_allclose(ours, ref, rtol=0, atol=1e-12)


def _keys(d):
    d = abs(d)
    a = Fraction(-1, 2)
    if d <= 1:
        return (a + 2) * d ** 3 - (a + 3) * d ** 2 + 1
    if d < 2:
        return a * d ** 3 - 5 * a * d ** 2 + 8 * a * d - 4 * a
    return Fraction(0)


def _exact(x, p, q, mode, pad, my, mx):
    H, W = len(x), len(x[0])

    def val(r, c):
        def rm(t, n):
            if 0 <= t < n:
                return t
            if pad == "zero":
                return None
            if pad == "replicate":
                return 0 if t < 0 else n - 1
            return -t if t < 0 else 2 * (n - 1) - t
        rr, cc = rm(r, H), rm(c, W)
        return Fraction(0) if rr is None or cc is None else Fraction(x[rr][cc])

    uy, ux = Fraction(my * q, p), Fraction(mx * q, p)
    by, bx = int(uy), int(ux)  # floor (non-negative)
    acc = Fraction(0)
    taps = {"nearest": [0], "bilinear": [0, 1], "bicubic": [-1, 0, 1, 2]}[mode]
    for a in taps:
        for c in taps:
            if mode == "nearest":
                w = 1
            elif mode == "bilinear":
                w = (1 - abs(uy - (by + a))) * (1 - abs(ux - (bx + c)))
            else:
                w = _keys(uy - (by + a)) * _keys(ux - (bx + c))
            acc += w * val(by + a, bx + c)
    return acc


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("pad", PADS)
def test_exact_rational_brute_force(mode, pad):
    rs = np.random.RandomState(11)
    H, W = 5, 6
    x = rs.randint(-9, 10, size=(H, W)).astype(np.float64)
    xi = x.astype(int).tolist()
    for (p, q) in [(3, 2), (5, 3), (3, 5), (7, 4)]:
        try:
            y = oracle.staged(x, p, q, mode, pad, floor_extent=False)
        except oracle.OracleError as e:
            # refused only when a kept output's last tap cannot be reflected back
            Ho = p * -(-H // q)
            last = ((Ho - 1) * q) // p + {"nearest": 0, "bilinear": 1, "bicubic": 2}[mode]
            assert pad == "reflect" and e.code == -2 and last > 2 * (H - 1)
            continue
        for my in range(y.shape[0]):
            for mx in range(y.shape[1]):
                e = _exact(xi, p, q, mode, pad, my, mx)
                assert abs(y[my, mx] - float(e)) <= 1e-12 * max(1.0, abs(float(e)))


def test_row_window_and_points_agree_with_whole_image():
    x = rng_input(12, (3, 40, 31)).astype(np.float32)
    for (p, q, mode, pad) in [(3, 5, "bicubic", "replicate"), (5, 3, "bicubic", "reflect"), (7, 5, "bilinear", "zero")]:
        full = oracle.staged(x, p, q, mode, pad, floor_extent=True)
        Ho = full.shape[1]
        r0, r1 = Ho // 3, (2 * Ho) // 3
        part = oracle.staged(x, p, q, mode, pad, floor_extent=True, rows=(r0, r1))
        np.testing.assert_array_equal(part, full[:, r0:r1])
        # the direct evaluator needs only the kept outputs' own taps ...
        lo_row = max(0, (r0 * q) // p - 1)
        hi_row = min(40, ((r1 - 1) * q) // p + 3)
        win = oracle.direct(x[:, lo_row:hi_row], p, q, mode, pad, floor_extent=True, rows=(r0, r1), H=40,
                            row0=lo_row)
        np.testing.assert_allclose(win, full[:, r0:r1], rtol=0, atol=1e-12)
        # ... the staged layer reads the whole window of every hidden row it computes
        lo_s = max(0, (r0 // p) * q - 1)
        hi_s = min(40, ((r1 - 1) // p) * q + ((p - 1) * q) // p + 3)
        win = oracle.staged(x[:, lo_s:hi_s], p, q, mode, pad, floor_extent=True, rows=(r0, r1), H=40, row0=lo_s)
        np.testing.assert_array_equal(win, full[:, r0:r1])
        pts = np.array([[1, 0, 0], [2, Ho - 1, full.shape[2] - 1], [0, r0, 3]])
        vals = oracle.direct_points(x, pts, p, q, mode, pad, floor_extent=True)
        np.testing.assert_allclose(vals, [full[1, 0, 0], full[2, Ho - 1, -1], full[0, r0, 3]], atol=1e-12)
        with pytest.raises(oracle.OracleError):  # a window that lacks needed rows is refused
            oracle.staged(x[:, lo_row + 3:hi_row], p, q, mode, pad, floor_extent=True, rows=(r0, r1), H=40,
                          row0=lo_row + 3)


def test_float32_input_path_equals_double():
    x = rng_input(13, (2, 12, 14)).astype(np.float32)
    a = oracle.staged(x, 5, 3, "bicubic", "reflect")
    b = oracle.staged(x.astype(np.float64), 5, 3, "bicubic", "reflect")
    np.testing.assert_array_equal(a, b)


def test_round_to_dtypes():
    import torch
    y = np.array([1.00390625, 1.01171875, 0.1, -2.5e-8, 65519.0, 1e30])
    bf = oracle.round_to(y, "bfloat16")
    # ties to even at bf16 precision (8 significand bits): 1+2^-8 -> 1, 1+3*2^-8 -> 1+2^-6
    assert bf[0].item() == 1.0 and bf[1].item() == 1.015625
    assert oracle.round_to(y, "float16")[4] == np.float16(65504.0)
    assert oracle.round_to(y, "float32").dtype == np.float32
    assert bf.dtype == torch.bfloat16


def test_empty_floor_extent_is_refused():
    x = rng_input(14, (5, 5))
    with pytest.raises(oracle.OracleError) as e:
        oracle.staged(x, 2, 11, "bilinear", "replicate", floor_extent=True)
    assert e.value.code == -3
