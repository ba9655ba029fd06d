"""Special values through the nearest-neighbour path, bit for bit.

§5.2.1 makes every nearest kernel a one-hot: each output
IS one (padded) input element.  The oracle cannot be the checker here -- it
multiplies the window by the one-hot (0 * Inf = NaN, -0 + 0 = +0, reading
Z11) -- so the pin is a plain index gather written in this file:
out[my][mx] = x~[floor(my q / p)][floor(mx q / p)] with x~ the padded input
(§3 Padding; zero pad = +0.0).  Inputs carry -0, +-Inf,
NaNs with payloads, subnormals and the largest finite values; every output's
bits must equal the gather's.  The fraction-0 outputs of bilinear/bicubic
(output rows and columns that are multiples of p) are exact copies too
(reading Z11): their bits are checked the same way (16-bit NaN payloads
excepted: that copy passes through fp32 registers).
"""
import itertools

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2203_10670_b200 import Plan

DEV = "cuda:0"
# special bit patterns per dtype: -0, +Inf, -Inf, quiet NaNs with payloads,
# a negative NaN, the smallest subnormal, -subnormal, the largest finite
SPECIALS = {
    "float32": (np.uint32, [0x80000000, 0x7F800000, 0xFF800000, 0x7FC01234, 0x7FFFFFFF, 0xFFC00001, 0x00000001,
                            0x80000001, 0x7F7FFFFF]),
    "float16": (np.uint16, [0x8000, 0x7C00, 0xFC00, 0x7E01, 0x7FFF, 0xFE02, 0x0001, 0x8001, 0x7BFF]),
    "bfloat16": (np.uint16, [0x8000, 0x7F80, 0xFF80, 0x7FC1, 0x7FFF, 0xFFC2, 0x0001, 0x8001, 0x7F7F]),
}
TORCH_INT = {"float32": torch.int32, "float16": torch.int16, "bfloat16": torch.int16}


def special_input(seed, shape, dtype):
    v = synth.normal_f32(seed, int(np.prod(shape))).reshape(shape)
    x = torch.from_numpy(v).to(getattr(torch, dtype)).contiguous()
    ut, pats = SPECIALS[dtype]
    bits = x.view(TORCH_INT[dtype]).numpy().view(ut).copy()
    rs = np.random.RandomState(seed)
    flat = bits.reshape(-1)
    idx = rs.choice(flat.size, size=flat.size // 3, replace=False)
    flat[idx] = np.array(pats, dtype=ut)[rs.randint(0, len(pats), idx.size)]
    flat[0] = pats[0]  # corners carry specials too
    flat[-1] = pats[3]
    return torch.from_numpy(bits.view(np.int32 if dtype == "float32" else np.int16)).view(getattr(torch, dtype))


def src_index(m, p, q, n, pad):
    """Source index of output m along a dimension of n inputs (nearest, floor);
    -1 for a zero-padding element."""
    s = (m * q) // p
    if s < n:
        return s
    if pad == "zero":
        return -1
    if pad == "replicate":
        return n - 1
    return 2 * (n - 1) - s  # reflect without edge repeat


def gather(bits, dims, odims, factors, pad):
    """out = x~[src(m_0), src(m_1), ...] over the trailing len(dims) axes (bits in, bits out)."""
    lead = bits.shape[: bits.ndim - len(dims)]
    idx = [np.array([src_index(m, p, q, n, pad) for m in range(no)]) for (p, q), n, no in zip(factors, dims, odims)]
    zero = np.zeros(1, dtype=bits.dtype)
    out = np.empty(lead + tuple(odims), dtype=bits.dtype)
    grids = np.meshgrid(*idx, indexing="ij")
    valid = np.ones(grids[0].shape, dtype=bool)
    for g in grids:
        valid &= g >= 0
    take = tuple(np.where(valid, g, 0) for g in grids)
    src = bits[(Ellipsis,) + take]
    out[...] = np.where(valid, src, zero[0])
    return out


@pytest.mark.parametrize("dtype", ["float32", "float16", "bfloat16"])
@pytest.mark.parametrize("W", [45, 48])
def test_nearest_special_values_bit_exact(dtype, W):
    """W = 48: 16-B rows (the row-staged kernel); W = 45: the general kernel."""
    ut = SPECIALS[dtype][0]
    n = 0
    for (p, q), pad, ext in itertools.product([(2, 3), (3, 4), (3, 2), (5, 3), (1, 1), (2, 1), (27, 11), (1, 4)],
                                              ["zero", "replicate", "reflect"], ["paper", "floor"]):
        n += 1
        x = special_input(100 + n, (2, 3, 29, W), dtype)
        pl = Plan(p, q, "nearest", pad, 3, 29, W, dtype, ext)
        assert pl.kernel == "nearest_gather"
        assert pl.launch_info(2)["variant"] in (("rows_staged", "rows_async") if W == 48 else ("general",))
        y = pl.run(x.to(DEV))
        got = y.cpu().view(TORCH_INT[dtype]).numpy().view(ut)
        exp = gather(x.view(TORCH_INT[dtype]).numpy().view(ut), (29, W), (pl.Ho, pl.Wo), [(pl.p, pl.q)] * 2, pad)
        assert np.array_equal(got, exp), f"{p}/{q} {pad} {ext} {dtype}: {int((got != exp).sum())} outputs differ"


def test_nearest_special_values_rank1_and_3d():
    for dtype in ("float32", "bfloat16"):
        ut = SPECIALS[dtype][0]
        x = special_input(7, (2, 2, 301), dtype)
        pl = Plan.nd([3], [5], "nearest", "replicate", 2, (301,), dtype, "paper")
        got = pl.run(x.to(DEV)).cpu().view(TORCH_INT[dtype]).numpy().view(ut)
        exp = gather(x.view(TORCH_INT[dtype]).numpy().view(ut), (301,), pl.odims, [(3, 5)], "replicate")
        assert np.array_equal(got, exp), dtype
        x = special_input(8, (1, 2, 5, 13, 17), dtype)
        pl = Plan.nd([2, 3, 5], [3, 2, 4], "nearest", "zero", 2, (5, 13, 17), dtype, "paper")
        got = pl.run(x.to(DEV)).cpu().view(TORCH_INT[dtype]).numpy().view(ut)
        exp = gather(x.view(TORCH_INT[dtype]).numpy().view(ut), (5, 13, 17), pl.odims, [(2, 3), (3, 2), (5, 4)],
                     "zero")
        assert np.array_equal(got, exp), dtype


@pytest.mark.parametrize("mode", ["bilinear", "bicubic"])
def test_fraction0_outputs_are_exact_copies(mode):
    """Outputs at phase (0, 0) read one input element with weight 1 (reading Z11):
    the fused kernel copies it, so specials pass through bit for bit."""
    for dtype, (p, q) in itertools.product(["float32", "float16", "bfloat16"], [(5, 3), (3, 2), (7, 5), (2, 3)]):
        ut = SPECIALS[dtype][0]
        x = special_input(300 + p * 10 + q, (1, 2, 40, 72), dtype)
        pl = Plan(p, q, mode, "replicate", 2, 40, 72, dtype, "floor")
        assert pl.kernel == "fused_separable"
        got = pl.run(x.to(DEV)).cpu().view(TORCH_INT[dtype]).numpy().view(ut)
        exp = gather(x.view(TORCH_INT[dtype]).numpy().view(ut), (40, 72), (pl.Ho, pl.Wo), [(p, q)] * 2, "replicate")
        sel = (slice(None), slice(None), slice(0, None, p), slice(0, None, p))
        g, e = got[sel], exp[sel]
        if dtype != "float32":
            # the copy goes through fp32 registers and the RNE store conversion
            # (cvt.rn.f16.f32 / cvt.rn.bf16x2.f32): every value and sign
            # survives, a NaN stays a NaN but its payload may not (Z11)
            em, mm = (0x7C00, 0x03FF) if dtype == "float16" else (0x7F80, 0x007F)
            nan_g = ((g & em) == em) & ((g & mm) != 0)
            nan_e = ((e & em) == em) & ((e & mm) != 0)
            assert np.array_equal(nan_g, nan_e), f"{mode} {p}/{q} {dtype}: NaN positions"
            g, e = g[~nan_e], e[~nan_e]
        assert np.array_equal(g, e), f"{mode} {p}/{q} {dtype}"


def test_nearest_row_kernel_equals_general_kernel(monkeypatch):
    """The row-staged gather and the general gather (FCFS_NO_NEAREST_ROWS) give
    the same bits on batches of jobs sharing one input: anisotropic factors,
    up- and down-scaling, paper extent rows past the last input row (reflect:
    rows read from global memory), several jobs in one launch."""
    import paper_2203_10670_b200 as fc
    for dtype in ("float32", "bfloat16"):
        x = special_input(11, (3, 2, 77, 96), dtype).to(DEV)
        plans = [Plan.nd(pq[0], pq[1], "nearest", pad, 2, (77, 96), dtype, ext)
                 for pq, pad, ext in [(((2, 3), (3, 4)), "zero", "floor"), (((5, 7), (3, 2)), "reflect", "paper"),
                                      (((3, 1), (4, 1)), "replicate", "paper"), (((1, 1), (1, 1)), "zero", "floor")]]
        for pl in plans:
            assert pl.launch_info(3)["variant"] in ("rows_staged", "rows_async")
        a = [torch.empty(pl.out_shape(3), dtype=x.dtype, device=DEV) for pl in plans]
        b = [torch.empty_like(t) for t in a]
        fc.run_batch([(pl, x, o) for pl, o in zip(plans, a)])
        torch.cuda.synchronize()
        monkeypatch.setenv("FCFS_NO_NEAREST_ROWS", "1")
        fc.run_batch([(pl, x, o) for pl, o in zip(plans, b)])
        torch.cuda.synchronize()
        monkeypatch.delenv("FCFS_NO_NEAREST_ROWS")
        for i, (u, v) in enumerate(zip(a, b)):
            assert torch.equal(u.view(TORCH_INT[dtype]), v.view(TORCH_INT[dtype])), (dtype, i)
