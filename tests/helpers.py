"""Comparison helpers for the parity tests (GPU result vs oracle)."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import synth

TOL_F32 = 1e-5  # max abs error relative to the input range (BASELINE.json north_star)


def ordered16(bits: np.ndarray) -> np.ndarray:
    """Map fp16/bf16 bit patterns to integers whose difference counts ulps."""
    b = bits.astype(np.int32) & 0xFFFF
    mag = b & 0x7FFF
    return np.where(b & 0x8000, -mag, mag)


def to_bits16(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().astype(np.int32) & 0xFFFF


WSUM = {"nearest": 1.0, "bilinear": 1.0, "bicubic": 1.25}  # max_f sum_t |w_t(f)| per dimension


def fp32_error_bound(mode: str, x_absmax: float) -> float:
    """Absolute error bound of the fp32 two-pass evaluation (<= 8 roundings of
    partial sums bounded by (sum|w|)^2 * max|x|): 2^-20 (sum|w|)^2 max|x|."""
    return 2.0 ** -20 * WSUM[mode] ** 2 * x_absmax


def compare(gpu: torch.Tensor, ref64: np.ndarray, dtype: str, mode: str, x_range: float, what: str = "",
            x_absmax: float | None = None):
    """Assert the BASELINE.json bar: nearest bit-exact; fp32 within 1e-5 * range;
    fp16/bf16 within 1 ulp of the oracle's fp32 result rounded to the dtype.

    Reading Z18: where the exact result lies so close to zero that
    the fp32 accumulation the bar prescribes cannot resolve 1 ulp of the dtype,
    an element also passes if |gpu - exact| <= 1 dtype-spacing + the fp32 error
    bound (fp32_error_bound).  The count of such elements is returned."""
    gpu = gpu.cpu()
    ref64 = np.asarray(ref64, dtype=np.float64).reshape(tuple(gpu.shape))
    if dtype == "float32":
        g = gpu.numpy().astype(np.float64)
        if mode == "nearest":
            np.testing.assert_array_equal(gpu.numpy().view(np.uint32), ref64.astype(np.float32).view(np.uint32),
                                          err_msg=what)
        else:
            err = np.abs(g - ref64).max() if g.size else 0.0
            assert err <= TOL_F32 * max(x_range, 1e-30), f"{what}: max abs err {err} > {TOL_F32} * {x_range}"
        return
    ref = oracle.round_to(ref64, dtype)
    ref_t = ref if isinstance(ref, torch.Tensor) else torch.from_numpy(ref)
    gb, rb = to_bits16(gpu), to_bits16(ref_t)
    if mode == "nearest":
        np.testing.assert_array_equal(gb, rb, err_msg=what)
        return
    d = np.abs(ordered16(gb) - ordered16(rb))
    bad = d > 1
    n_near_zero = 0
    if bad.any():
        xa = x_range if x_absmax is None else x_absmax
        g64 = gpu.to(torch.float64).numpy()
        nxt = torch.from_numpy(((rb + 1) & 0xFFFF).astype(np.int16).view(np.int16)).view(ref_t.dtype)
        spacing = np.abs(nxt.to(torch.float64).numpy() - ref_t.to(torch.float64).numpy())
        ok2 = np.abs(g64 - ref64) <= spacing + fp32_error_bound(mode, xa)
        n_near_zero = int((bad & ok2).sum())
        bad &= ~ok2
    assert not bad.any(), (f"{what}: {int(d[bad].max())} ulp at {np.unravel_index(np.argmax(np.where(bad, d, -1)), d.shape)}"
                           f" gpu={gpu.flatten()[np.argmax(np.where(bad, d, -1))]} exact="
                           f"{ref64.flatten()[np.argmax(np.where(bad, d, -1))]}")
    return n_near_zero


def oracle_input(x_cpu: torch.Tensor) -> np.ndarray:
    """Exact fp32 image of the input values for the oracle (fp16/bf16 -> fp32 is exact)."""
    return x_cpu.float().numpy()


def sample_points(rs: np.random.RandomState, planes: int, Ho: int, Wo: int, n: int) -> np.ndarray:
    """Random outputs plus every corner and the first/last rows and columns of a few planes."""
    pts = [np.stack([rs.randint(0, planes, n), rs.randint(0, Ho, n), rs.randint(0, Wo, n)], 1)]
    for pl in sorted({0, planes - 1, planes // 2}):
        cols = np.arange(Wo)
        rows = np.arange(Ho)
        for r in (0, 1, Ho - 2, Ho - 1):
            if 0 <= r < Ho:
                pts.append(np.stack([np.full(Wo, pl), np.full(Wo, r), cols], 1))
        for c in (0, 1, Wo - 2, Wo - 1):
            if 0 <= c < Wo:
                pts.append(np.stack([np.full(Ho, pl), rows, np.full(Ho, c)], 1))
    return np.concatenate(pts).astype(np.int64)


def make_cfg_input(cfg: synth.Config, n1=None):
    return synth.make_input(cfg, 0, n1)
