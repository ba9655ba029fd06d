"""Race and coverage checks of the asynchronous pipelines.

compute-sanitizer (racecheck / synccheck / memcheck) is closed on the GPU
pool these tests run on (runs under it have left GPUs needing a reset), so
the hazards it would look for are provoked and detected directly:

* coverage -- every output buffer is pre-filled with a NaN pattern no
  finite input can produce; after the run no element may still hold it (a
  store skipped by a lost mbarrier phase or a mis-sized bulk copy would);
* determinism under re-timing -- each kernel runs under launch geometries
  that change its pipeline timing: ring depth (FCFS_DEBUG_S = 2: the
  producer waits on every stage), grid size (one CTA: every task in one
  pipeline; 7 CTAs: uneven task counts), band split, flush groups, TMA box
  vs row copies, programmatic launch off, and the nearest row ring's depth.
  A missing barrier or wrong phase parity shows up as results that differ
  between schedules; every schedule must give the default run's bits;
* repetition -- the same launch five times, bitwise identical (the weight
  gradient accumulates with atomics: compared within its Z22 bound instead).

The outputs are checked against the oracle elsewhere (test_gpu_parity,
test_gpu_variants); here the default run is the reference of every other.
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2203_10670_b200 as fc
    from paper_2203_10670_b200 import Plan

DEV = "cuda:0"
POISON = {torch.float32: 0x7FC0BEEF, torch.float16: 0x7E5A, torch.bfloat16: 0x7FDA}
IV = {torch.float32: torch.int32, torch.float16: torch.int16, torch.bfloat16: torch.int16}


def poisoned(shape, dtype):
    """A buffer of a NaN pattern (quiet NaN with a payload) that no finite input produces."""
    t = torch.empty(shape, dtype=dtype, device=DEV)
    t.view(IV[dtype]).fill_(POISON[dtype])
    return t


def no_poison(t):
    return not bool((t.view(IV[t.dtype]) == POISON[t.dtype]).any())


def x_of(shape, dtype, seed):
    return torch.from_numpy(synth.normal_f32(seed, int(np.prod(shape))).reshape(shape)).to(dtype).to(DEV)


FORWARD_SCHEDULES = [{}, {"FCFS_DEBUG_S": "2"}, {"FCFS_DEBUG_GRID": "1"}, {"FCFS_DEBUG_GRID": "7"},
                     {"FCFS_DEBUG_NBANDS": "1"}, {"FCFS_DEBUG_NBANDS": "9"}, {"FCFS_DEBUG_G": "1"},
                     {"FCFS_DEBUG_G": "2"}, {"FCFS_NO_TMA": "1"}, {"FCFS_NO_PDL": "1"},
                     {"FCFS_DEBUG_S": "2", "FCFS_DEBUG_GRID": "3", "FCFS_NO_TMA": "1"}]


def run_forward(pl, x, N):
    out = poisoned(pl.out_shape(N), x.dtype)
    pl.run(x, out=out)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("case", [
    # (p, q, mode, pad, N, C, H, W, dtype): fused aligned / column tiles / unaligned rows (sw_load) / tiled / 3-deep
    (5, 3, "bicubic", "reflect", 3, 4, 61, 128, torch.bfloat16),
    (7, 5, "bilinear", "replicate", 1, 2, 97, 1200, torch.float16),
    (3, 5, "bicubic", "replicate", 1, 1, 301, 2048, torch.float32),
    (5, 3, "bicubic", "zero", 2, 3, 45, 37, torch.bfloat16),
    (4, 7, "bilinear", "reflect", 2, 2, 77, 250, torch.float16),
    (27, 11, "bicubic", "replicate", 1, 2, 70, 90, torch.float32),
])
def test_forward_schedules_identical_and_complete(case, monkeypatch):
    p, q, mode, pad, N, C, H, W, dtype = case
    pl = Plan(p, q, mode, pad, C, H, W, {torch.float32: "float32", torch.float16: "float16",
                                         torch.bfloat16: "bfloat16"}[dtype], "floor")
    x = x_of((N, C, H, W), dtype, 31 + p * 7 + q)
    ref = None
    for env in FORWARD_SCHEDULES:
        for k in ("FCFS_DEBUG_S", "FCFS_DEBUG_GRID", "FCFS_DEBUG_NBANDS", "FCFS_DEBUG_G", "FCFS_NO_TMA", "FCFS_NO_PDL"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        y = run_forward(pl, x, N)
        assert no_poison(y), (case, env, "an output was never written")
        if ref is None:
            ref = y
        else:
            assert torch.equal(y.view(IV[dtype]), ref.view(IV[dtype])), (case, env)
    for k in ("FCFS_DEBUG_S", "FCFS_DEBUG_GRID", "FCFS_DEBUG_NBANDS", "FCFS_DEBUG_G", "FCFS_NO_TMA", "FCFS_NO_PDL"):
        monkeypatch.delenv(k, raising=False)
    for _ in range(5):  # the same schedule, again
        assert torch.equal(run_forward(pl, x, N).view(IV[dtype]), ref.view(IV[dtype])), case


def test_nearest_row_ring_schedules(monkeypatch):
    """The row gathers (async and staged) under every ring depth and grid: same bits, no gaps."""
    x = x_of((4, 3, 200, 256), torch.float32, 5)
    plans = [Plan(2, 3, "nearest", "zero", 3, 200, 256, "float32", "floor"),
             Plan(3, 4, "nearest", "zero", 3, 200, 256, "float32", "floor"),
             Plan(7, 5, "nearest", "reflect", 3, 200, 256, "float32", "paper")]
    ref = None
    # default: the async row kernel (two row buffers per warp); FCFS_NEAREST_STAGED: the
    # producer-warp kernel with its slot rings
    st = {"FCFS_NEAREST_STAGED": "1"}
    for env in [{}, {"FCFS_DEBUG_NEAREST_GRID": "1"}, {"FCFS_DEBUG_NEAREST_GRID": "5"},
                {"FCFS_DEBUG_NEAREST_CTAS": "1"}, {"FCFS_NO_PDL": "1"},
                st, {**st, "FCFS_DEBUG_NEAREST_LOG2SW": "0"}, {**st, "FCFS_DEBUG_NEAREST_LOG2SW": "1"},
                {**st, "FCFS_DEBUG_NEAREST_GRID": "1"}, {**st, "FCFS_DEBUG_NEAREST_GRID": "5"},
                {**st, "FCFS_DEBUG_NEAREST_CTAS": "2"}]:
        for k in ("FCFS_DEBUG_NEAREST_LOG2SW", "FCFS_DEBUG_NEAREST_GRID", "FCFS_NO_PDL", "FCFS_DEBUG_NEAREST_CTAS",
                  "FCFS_NEAREST_STAGED"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        outs = [poisoned(pl.out_shape(4), torch.float32) for pl in plans]
        fc.run_batch([(pl, x, o) for pl, o in zip(plans, outs)])
        torch.cuda.synchronize()
        for o in outs:
            assert no_poison(o), env
        if ref is None:
            ref = outs
        else:
            for a, b in zip(outs, ref):
                assert torch.equal(a.view(torch.int32), b.view(torch.int32)), env


def test_adjoint_schedules(monkeypatch):
    """Fused adjoint + border bands (two launches, the second rewriting bands
    the first wrote) under different schedules: same bits, no gaps."""
    pl = Plan(5, 3, "bicubic", "reflect", 3, 61, 128, "bfloat16", "floor")
    g = x_of(pl.out_shape(2), torch.bfloat16, 9)
    ref = None
    for env in [{}, {"FCFS_DEBUG_S": "2"}, {"FCFS_DEBUG_GRID": "1"}, {"FCFS_DEBUG_BAND_TH": "4"},
                {"FCFS_DEBUG_BAND_PB": "1"}, {"FCFS_NO_PDL": "1"}, {"FCFS_NO_FUSED_ADJOINT": "1"}]:
        for k in ("FCFS_DEBUG_S", "FCFS_DEBUG_GRID", "FCFS_DEBUG_BAND_TH", "FCFS_DEBUG_BAND_PB", "FCFS_NO_PDL",
                  "FCFS_NO_FUSED_ADJOINT"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        out = poisoned(pl.in_shape(2), torch.bfloat16)
        pl.run_adjoint(g, out=out)
        torch.cuda.synchronize()
        assert no_poison(out), env
        if ref is None:
            ref = out
        elif "FCFS_NO_FUSED_ADJOINT" not in env:  # (the tiled kernel sums in another order)
            assert torch.equal(out.view(torch.int16), ref.view(torch.int16)), env


def test_weight_gradient_repeatable():
    """Atomic accumulation: repeated runs agree within the Z22 bound and are complete."""
    pl = Plan(5, 3, "bicubic", "reflect", 4, 64, 64, "float32", "floor")
    x = x_of((2, 4, 64, 64), torch.float32, 3)
    g = x_of(pl.out_shape(2), torch.float32, 4)
    outs = [pl.run_weight_grad(x, g) for _ in range(5)]
    torch.cuda.synchronize()
    bound = (g.numel() + 8) * 2.0 ** -24 * float((g.abs().sum() * x.abs().max()).item())
    for o in outs:
        assert torch.isfinite(o).all()
        assert float((o - outs[0]).abs().max()) <= bound
