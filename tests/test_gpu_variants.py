"""Every compiled fused variant against the oracle -- generated from the
variant tables themselves (csrc/fused_pairs.h), so a pair added there is
tested here without editing this file.

For each table (isotropic 2D, width-only, height-only, 3D, adjoint) x
{bilinear, bicubic} x {float32, float16, bfloat16} x {zero, replicate,
reflect}: a ragged shape (rows and columns not a multiple of the period,
several tiles for the wide one), every output compared with the staged
oracle at the BASELINE.json bar (oracle.staged / staged_nd / adjoint_nd,
pinned in test_oracle_*_pins.py), bitwise equality with the reference
kernel, and fcfs_launch_info / fcfs_adjoint_info asserting that the variant
under test is the kernel that ran.  Forward: PAPER.md:106-116 (§3.1) and
:154-167 (§4.2); weights §5.2.2-3; adjoint: DESIGN.md Z21.
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
DTYPES = ["float32", "float16", "bfloat16"]
PADS = ["zero", "replicate", "reflect"]
MODES = ["bilinear", "bicubic"]
ESZ = {"float32": 4, "float16": 2, "bfloat16": 2}


def table_pairs(macro: str):
    """The (p, q) pairs listed by `#define <macro>(Y) Y(p, q) ...` in fused_pairs.h."""
    src = open(PAIRS_H).read()
    m = re.search(r"#define\s+" + macro + r"\(Y\)((?:[^\n]*\\\n)*[^\n]*)", src)
    assert m, macro
    pairs = [(int(a), int(b)) for a, b in re.findall(r"Y\((\d+),\s*(\d+)\)", m.group(1))]
    assert pairs, macro
    return pairs


ISO = table_pairs("FCFS_ISO_PAIRS")
NONUNIT = table_pairs("FCFS_NONUNIT_PAIRS")
ZPAIRS = table_pairs("FCFS_Z_PAIRS")
# ragged shapes (H, W): W keeps rows 16-B aligned for every dtype (the aligned
# producer path); the wide one splits rows into column tiles
SHAPES = [(37, 72), (29, 520), (53, 136)]
SLICE_FACTORS = [(3, 2), (2, 3), (5, 3), (1, 2), (4, 3)]


def make_x(seed, shape, dtype):
    v = synth.normal_f32(seed, int(np.prod(shape))).reshape(shape)
    return torch.from_numpy(v).to(getattr(torch, dtype))


def _check_forward(x, p, q, mode, pad, dtype, extent, what, expect):
    pl = Plan.nd(p, q, mode, pad, x.shape[1], tuple(x.shape[2:]), dtype, extent)
    info = pl.launch_info(x.shape[0])
    assert info["kernel"] == "fused_separable", (what, info)
    for k, v in expect.items():
        assert v(info[k]) if callable(v) else info[k] == v, (what, k, info)
    y = pl.run(x.to(DEV))
    torch.cuda.synchronize()
    xr = oracle_input(x)
    ref = oracle.staged_nd(xr, list(p), list(q), mode, pad, floor_extent=extent == "floor")
    assert tuple(y.shape) == ref.shape, what
    n = compare(y, ref, dtype, mode, float(xr.max() - xr.min()), what, x_absmax=float(np.abs(xr).max()))
    yr = Plan.nd(p, q, mode, pad, x.shape[1], tuple(x.shape[2:]), dtype, extent, force_reference=True).run(x.to(DEV))
    assert torch.equal(y.view(torch.uint8), yr.view(torch.uint8)), f"{what}: fused != reference kernel"
    return n


def _cases(pairs):
    for i, ((P, Q), mode, dtype) in enumerate(itertools.product(pairs, MODES, DTYPES)):
        yield i, P, Q, mode, dtype


@pytest.mark.parametrize("pad", PADS)
def test_isotropic_variants(pad):
    n_relaxed = 0
    for i, P, Q, mode, dtype in _cases(ISO):
        H, W = SHAPES[i % len(SHAPES)]
        ext = ["floor", "paper"][i % 2]
        x = make_x(5000 + i, (2, 2, H, W), dtype)
        n_relaxed += _check_forward(x, (P, P), (Q, Q), mode, pad, dtype, ext, f"iso {P}/{Q} {mode} {pad} {dtype}",
                                    {"PY": P, "QY": Q, "PX": P, "QX": Q, "TZ": 1})
    print(f"isotropic variants ({pad}): {n_relaxed} relaxed elements")


@pytest.mark.parametrize("pad", PADS)
def test_width_only_variants(pad):
    for i, P, Q, mode, dtype in _cases(NONUNIT):
        H, W = SHAPES[(i + 1) % len(SHAPES)]
        ext = ["paper", "floor"][i % 2]
        x = make_x(6000 + i, (1, 3, H, W), dtype)
        # rows 1/1 run as an unreduced identity R/R (every row phase a copy)
        _check_forward(x, (1, P), (1, Q), mode, pad, dtype, ext, f"W {P}/{Q} {mode} {pad} {dtype}",
                       {"PX": P, "QX": Q, "TZ": 1, "PY": lambda v: v >= 1, "QY": lambda v: v >= 1})


@pytest.mark.parametrize("pad", PADS)
def test_height_only_variants(pad, monkeypatch):
    # the row-pipelined kernel's identity-column variants (the height-only row
    # kernel, which takes these aligned shapes by default, has its own table
    # test: test_gpu_vpass.py)
    monkeypatch.setenv("FCFS_NO_VPASS", "1")
    for i, P, Q, mode, dtype in _cases(NONUNIT):
        H, W = SHAPES[(i + 2) % len(SHAPES)]
        ext = ["floor", "paper"][i % 2]
        x = make_x(7000 + i, (2, 1, H, W), dtype)
        _check_forward(x, (P, 1), (Q, 1), mode, pad, dtype, ext, f"H {P}/{Q} {mode} {pad} {dtype}",
                       {"PY": P, "QY": Q, "TZ": 1})


@pytest.mark.parametrize("pad", PADS)
def test_volume_variants(pad, monkeypatch):
    # the row-pipelined 3D variants (the slice-ring plane kernel, which takes most
    # of these volumes by default, has its own table test: test_gpu_plane3.py)
    monkeypatch.setenv("FCFS_NO_PLANE3", "1")
    for i, P, Q, mode, dtype in _cases(ZPAIRS):
        pz, qz = SLICE_FACTORS[i % len(SLICE_FACTORS)]
        ext = ["floor", "paper"][i % 2]
        x = make_x(8000 + i, (1, 2, 7, 23, 40), dtype)
        _check_forward(x, (pz, P, P), (qz, Q, Q), mode, pad, dtype, ext,
                       f"3D {pz}/{qz} x {P}/{Q} {mode} {pad} {dtype}",
                       {"PY": P, "QY": Q, "PX": P, "QX": Q, "TZ": lambda v: v > 1})


def test_unaligned_rows_every_variant():
    """Odd widths (rows not 16-B aligned: the in-place shifted reads) for every
    isotropic variant and mode, cycling dtype and pad."""
    for i, P, Q, mode, _ in _cases(ISO):
        dtype, pad = DTYPES[i % 3], PADS[(i // 3) % 3]
        x = make_x(9000 + i, (1, 3, 31, 37), dtype)
        _check_forward(x, (P, P), (Q, Q), mode, pad, dtype, "floor", f"odd-W {P}/{Q} {mode} {pad} {dtype}",
                       {"PY": P, "QY": Q, "PX": P, "QX": Q})


def _adjoint_fused_expected(P, Q, mode, dtype):
    """The adjoint variant is compiled usable (FusedVariant::ok) when A^T's first
    tap offset fits the stage's left margin of 16 B (fused_inst.cuh)."""
    T0, LO0 = (4, -1) if mode == "bicubic" else (2, 0)
    lo = -((-(1 - LO0 - T0) * P) // Q)  # ceil((1 - LO0 - T0) * P / Q)
    return -lo <= 16 // ESZ[dtype]


@pytest.mark.parametrize("pad", PADS)
def test_adjoint_variants(pad):
    from test_gpu_adjoint import run_adjoint_case
    for i, P, Q, mode, dtype in _cases(NONUNIT):
        H, W = SHAPES[i % len(SHAPES)]
        ext = ["floor", "paper"][i % 2]
        pl = Plan.nd((P, P), (Q, Q), mode, pad, 2, (H, W), dtype, ext)
        info = pl.adjoint_info(2)
        if _adjoint_fused_expected(P, Q, mode, dtype):
            assert info["kernel"] == "fused_adjoint", (P, Q, mode, dtype, pad, info)
            assert (info["PX"], info["QX"]) == (P, Q), info
            if pad == "zero":  # zero padding has no padding images to fold back
                assert info["bands"] == 0 and info["launches"] == 1, info
        else:
            assert info["kernel"] == "tiled_adjoint", (P, Q, mode, dtype, pad, info)
        run_adjoint_case((H, W), (P, P), (Q, Q), mode, pad, dtype, N=2, C=2, extent=ext, seed=10000 + i)
