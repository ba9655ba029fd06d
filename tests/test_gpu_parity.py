"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bar (BASELINE.json north_star): nearest bit-exact; fp32 max abs error <=
1e-5 x input range; fp16/bf16 within 1 ulp of the oracle's fp32 result rounded
to the dtype.  Full-size configs are checked on sampled outputs (plus whole
border rows/columns) computed one by one by the oracle's direct evaluator, on
every output by the staged oracle (in chunks of planes), and on every output
against the reference kernel (bitwise: both kernels share one arithmetic contract).
"""
import itertools
import zlib

import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import compare, oracle_input, sample_points

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2203_10670_b200 as fc
    from paper_2203_10670_b200 import Plan
    from paper_2203_10670_b200._lib import FcfsError

DEV = "cuda:0"


def run_cfg(cfg: synth.Config, x_dev, force_reference=False):
    pl = Plan(cfg.p, cfg.q, cfg.mode, cfg.pad, cfg.C, cfg.H, cfg.W, cfg.dtype,
              "floor" if cfg.floor_extent else "paper", cfg.is1d, force_reference=force_reference)
    y = pl.run(x_dev)
    torch.cuda.synchronize()
    return pl, y


def check_full_config(cfg: synth.Config, n_points=60000, chunk_planes=256):
    """Every output of a BASELINE config against the staged oracle (in chunks of
    planes), sampled outputs against the direct evaluator, and every output
    against the reference kernel (bitwise).  Returns (plan, relaxed Z18 count)."""
    x = synth.make_input(cfg)
    xd = x.to(DEV)
    pl, y = run_cfg(cfg, xd)
    xr = oracle_input(x)
    rng = float(xr.max() - xr.min())
    amax = float(np.abs(xr).max())
    planes = cfg.planes
    Ho, Wo = pl.output_shape()
    assert tuple(y.shape) == (cfg.N, cfg.C, Ho, Wo)
    ext = dict(floor_extent=cfg.floor_extent, is1d=cfg.is1d)
    # (1) sampled outputs, direct evaluator, one by one
    rs = np.random.RandomState(cfg.seed % 1000)
    pts = sample_points(rs, planes, Ho, Wo, n_points)
    ref = oracle.direct_points(xr.reshape(planes, cfg.H, cfg.W), pts, cfg.p, cfg.q, cfg.mode, cfg.pad, **ext)
    got = y.reshape(planes, Ho, Wo)[torch.from_numpy(pts[:, 0]), torch.from_numpy(pts[:, 1]),
                                    torch.from_numpy(pts[:, 2])]
    compare(got, ref, cfg.dtype, cfg.mode, rng, f"{cfg.name} sampled", x_absmax=amax)
    # (2) every output, staged oracle (all outputs of C1-C4)
    yc = y.reshape(planes, Ho, Wo).cpu()
    xp = xr.reshape(planes, cfg.H, cfg.W)
    relaxed = 0
    for p0 in range(0, planes, chunk_planes):
        p1 = min(planes, p0 + chunk_planes)
        ref = oracle.staged(xp[p0:p1], cfg.p, cfg.q, cfg.mode, cfg.pad, **ext)
        relaxed += compare(yc[p0:p1], ref, cfg.dtype, cfg.mode, rng, f"{cfg.name} planes {p0}:{p1}", x_absmax=amax)
    print(f"{cfg.name}: every output ({planes * Ho * Wo}) checked against the oracle, {relaxed} relaxed (Z18)")
    # (3) every output: fused/gather kernel == reference kernel, bitwise
    _, yr = run_cfg(cfg, xd, force_reference=True)
    assert torch.equal(y.view(torch.int16 if cfg.dtype != "float32" else torch.int32),
                       yr.view(torch.int16 if cfg.dtype != "float32" else torch.int32)), f"{cfg.name}: kernels differ"
    return pl, relaxed


@pytest.mark.parametrize("name", ["C1a", "C1b"])
def test_config1_every_output(name):
    cfg = synth.CONFIGS[name]
    x = synth.make_input(cfg)
    pl, y = run_cfg(cfg, x.to(DEV))
    ref = oracle.staged(oracle_input(x), cfg.p, cfg.q, cfg.mode, cfg.pad, floor_extent=cfg.floor_extent,
                        is1d=cfg.is1d)
    compare(y, ref, cfg.dtype, cfg.mode, float(x.max() - x.min()), name, x_absmax=float(x.abs().max()))
    assert tuple(y.shape[-2:]) == {"C1a": (72, 96), "C1b": (1, 67)}[name]


@pytest.mark.parametrize("name", ["C2a", "C2b"])
def test_config2_nearest_bit_exact_every_output(name):
    cfg = synth.CONFIGS[name]
    x = synth.make_input(cfg)
    pl, y = run_cfg(cfg, x.to(DEV))
    assert pl.kernel == "nearest_gather"
    ref = oracle.staged(oracle_input(x), cfg.p, cfg.q, cfg.mode, cfg.pad, floor_extent=True)
    compare(y, ref, cfg.dtype, cfg.mode, 1.0, name)


def test_config3_bicubic_bf16():
    pl, relaxed = check_full_config(synth.CONFIGS["C3"])
    assert relaxed <= 1e-5 * 4096 * 213 * 213
    assert pl.kernel == "fused_separable" and pl.output_shape() == (213, 213)


@pytest.mark.parametrize("name", ["C4a", "C4b"])
def test_config4_bilinear_fp16(name):
    pl, relaxed = check_full_config(synth.CONFIGS[name], chunk_planes=4)
    assert pl.kernel == "fused_separable"


def test_config5_giant_image_every_output():
    cfg = synth.CONFIGS["C5"]
    x = synth.make_input(cfg)
    xd = x.to(DEV)
    pl, y = run_cfg(cfg, xd)
    assert pl.kernel == "fused_separable" and pl.output_shape() == (19660, 19660)
    xr = x.numpy()
    rng = float(xr.max() - xr.min())
    rs = np.random.RandomState(5)
    pts = sample_points(rs, 1, 19660, 19660, 100000)
    ref = oracle.direct_points(xr.reshape(1, cfg.H, cfg.W), pts, cfg.p, cfg.q, cfg.mode, cfg.pad, floor_extent=True)
    got = y.reshape(19660, 19660)[torch.from_numpy(pts[:, 1]), torch.from_numpy(pts[:, 2])]
    compare(got, ref, "float32", "bicubic", rng, "C5 sampled")
    # every output row within +-4 of each 8-way strip boundary
    rows = []
    for g in range(1, 8):
        o0, o1, n0, n1 = pl.strip_rows(g * 4096, (g + 1) * 4096)
        rows += list(range(max(0, o0 - 4), min(19660, o0 + 5)))
    r = np.array(sorted(set(rows)))
    for r0 in r:
        lo = max(0, (r0 * 5) // 3 - 2)
        hi = min(cfg.H, (r0 * 5) // 3 + 4)
        ref = oracle.direct(xr[0, 0, lo:hi], 3, 5, "bicubic", "replicate", floor_extent=True, rows=(r0, r0 + 1),
                            H=cfg.H, row0=lo)
        compare(y[0, 0, r0:r0 + 1], ref, "float32", "bicubic", rng, f"C5 row {r0}")
    # every output, staged oracle in blocks of output rows (all C5
    # outputs when host RAM allows; the image is never padded whole in double)
    yc = y.reshape(19660, 19660).cpu().numpy()
    for r0 in range(0, 19660, 2048):
        r1 = min(19660, r0 + 2048)
        # the staged layer's union window of hidden positions i = m div 3: rows [5i - 1, 5i + 5]
        n0, n1 = max(0, 5 * (r0 // 3) - 1), min(cfg.H, 5 * ((r1 - 1) // 3) + 6)
        ref = oracle.staged(xr[0, 0, n0:n1], cfg.p, cfg.q, cfg.mode, cfg.pad, floor_extent=True, rows=(r0, r1),
                            H=cfg.H, row0=n0)
        err = float(np.abs(yc[r0:r1].astype(np.float64) - ref).max())
        assert err <= 1e-5 * rng, f"C5 rows {r0}:{r1}: max abs err {err}"
    # every output: fused == reference, bitwise
    _, yr = run_cfg(cfg, xd, force_reference=True)
    assert torch.equal(y.view(torch.int32), yr.view(torch.int32))


FACTORS = [(1, 1), (3, 2), (2, 3), (5, 3), (3, 5), (7, 5), (4, 7), (2, 1), (1, 2), (4, 3), (5, 4), (2, 11),
           (27, 11), (6, 5), (3, 4)]
DTYPES = ["float32", "float16", "bfloat16"]


def _rand_input(seed, shape, dtype):
    v = synth.normal_f32(seed, int(np.prod(shape))).reshape(shape)
    return torch.from_numpy(v).to(getattr(torch, dtype))


@pytest.mark.parametrize("mode", ["nearest", "bilinear", "bicubic"])
@pytest.mark.parametrize("pad", ["zero", "replicate", "reflect"])
def test_sweep_every_output(mode, pad):
    """Small ragged shapes spanning several tiles, every factor/dtype/extent: all outputs."""
    rs = np.random.RandomState(zlib.crc32(f"{mode}-{pad}".encode()))
    n = 0
    for (p, q), dtype in itertools.product(FACTORS, DTYPES):
        H = int(rs.randint(3, 90))
        W = int(rs.choice([8, 16, 24, 40, 64, 72, 96, 104, 120, 200, 264, 328, 37, 101]))
        N, C = int(rs.randint(1, 3)), int(rs.randint(1, 4))
        ext = ["paper", "floor"][n % 2]
        n += 1
        x = _rand_input(1000 + n, (N, C, H, W), dtype)
        try:
            pl = Plan(p, q, mode, pad, C, H, W, dtype, ext)
        except FcfsError as e:
            with pytest.raises(oracle.OracleError):
                oracle.staged(oracle_input(x), p, q, mode, pad, floor_extent=(ext == "floor"))
            assert e.name in ("FCFS_E_PAD", "FCFS_E_SHAPE")
            continue
        y = pl.run(x.to(DEV))
        torch.cuda.synchronize()
        xr = oracle_input(x)
        ref = oracle.staged(xr, p, q, mode, pad, floor_extent=(ext == "floor"))
        compare(y, ref, dtype, mode, float(xr.max() - xr.min()), f"{p}/{q} {mode} {pad} {dtype} {ext} {H}x{W}",
                x_absmax=float(np.abs(xr).max()))
        yr = Plan(p, q, mode, pad, C, H, W, dtype, ext, force_reference=True).run(x.to(DEV))
        assert torch.equal(y.cpu().view(torch.uint8), yr.cpu().view(torch.uint8)), f"{p}/{q} {mode} {pad} kernels"


@pytest.mark.parametrize("mode", ["nearest", "bilinear", "bicubic"])
def test_1d_rows(mode):
    for (p, q), dtype in itertools.product([(2, 3), (3, 2), (5, 3), (27, 11)], DTYPES):
        x = _rand_input(7, (2, 3, 5, 101), dtype)
        pl = Plan(p, q, mode, "replicate", 3, 5, 101, dtype, "floor", is1d=True)
        y = pl.run(x.to(DEV))
        ref = oracle.staged(oracle_input(x), p, q, mode, "replicate", floor_extent=True, is1d=True)
        compare(y, ref, dtype, mode, float(x.float().max() - x.float().min()), f"1d {p}/{q} {dtype}",
                x_absmax=float(x.float().abs().max()))


def test_identity_bit_exact():
    for mode, pad, dtype in itertools.product(["nearest", "bilinear", "bicubic"], ["zero", "replicate", "reflect"],
                                              DTYPES):
        x = _rand_input(3, (2, 3, 33, 64), dtype).to(DEV)
        y = fc.scale(x, 3, 3, mode, pad)
        assert torch.equal(y.view(torch.int16 if dtype != "float32" else torch.int32),
                           x.view(torch.int16 if dtype != "float32" else torch.int32))


def test_pixel_repetition():
    x = _rand_input(4, (1, 2, 21, 40), "float32").to(DEV)
    for p in (2, 3, 4):
        y = fc.scale(x, p, 1, "nearest", "zero")
        ref = x.repeat_interleave(p, dim=2).repeat_interleave(p, dim=3)
        assert torch.equal(y, ref)


def test_strips_equal_whole_image():
    """Row strips run one after another on one GPU (halo rows sliced from the
    whole input) reproduce the single-launch output bit for bit."""
    for (p, q, mode, pad, dtype) in [(3, 5, "bicubic", "replicate", "float32"), (5, 3, "bicubic", "reflect", "bfloat16"),
                                     (7, 5, "bilinear", "zero", "float16"), (2, 3, "nearest", "zero", "float32"),
                                     (4, 7, "bilinear", "replicate", "float16")]:
        H, W = 997, 640
        x = _rand_input(9, (1, 2, H, W), dtype).to(DEV)
        pl = Plan(p, q, mode, pad, 2, H, W, dtype, "floor")
        whole = pl.run(x)
        for G in (2, 3, 8):
            parts = []
            for g in range(G):
                own0, own1 = g * H // G, (g + 1) * H // G
                o0, o1, n0, n1 = pl.strip_rows(own0, own1)
                local = x[:, :, n0:n1].contiguous()
                parts.append(pl.run_rows(local, n0, o0, o1 - o0))
                if o1 > o0 and n1 - n0 > 1:  # a window without its first halo row is refused
                    with pytest.raises(FcfsError) as e:
                        pl.run_rows(x[:, :, n0 + 1:n1].contiguous(), n0 + 1, o0, o1 - o0)
                    assert e.value.name == "FCFS_E_SHAPE"
            got = torch.cat(parts, dim=2)
            assert torch.equal(got.view(torch.uint8), whole.view(torch.uint8)), f"{p}/{q} {mode} G={G}"


def test_misaligned_and_odd_pitch_buffers():
    # an input view offset by one element defeats 16-B bulk copies: the plan must
    # still be correct (reference kernel), and odd W too.
    for dtype in DTYPES:
        base = _rand_input(5, (1 * 2 * 50 * 64 + 1,), dtype).to(DEV)
        x = base[1:].view(1, 2, 50, 64)
        pl = Plan(5, 3, "bicubic", "reflect", 2, 50, 64, dtype, "floor")
        y = pl.run(x)
        ref = oracle.staged(oracle_input(x.cpu()), 5, 3, "bicubic", "reflect", floor_extent=True)
        compare(y, ref, dtype, "bicubic", float(x.float().max() - x.float().min()), f"misaligned {dtype}",
                x_absmax=float(x.float().abs().max()))
        out_base = torch.empty(y.numel() + 1, dtype=y.dtype, device=DEV)
        y2 = out_base[1:].view(y.shape)
        pl.run(x, out=y2)
        assert torch.equal(y2.view(torch.uint8), y.view(torch.uint8))


def test_edge_shapes():
    for (N, C, H, W) in [(1, 1, 1, 1), (1, 1, 1, 8), (1, 1, 2, 2), (3, 1, 7, 5), (1, 1, 300, 8), (1, 1, 2, 2048)]:
        for mode, pad in itertools.product(["nearest", "bilinear", "bicubic"], ["zero", "replicate", "reflect"]):
            x = _rand_input(6, (N, C, H, W), "float32")
            try:
                pl = Plan(5, 3, mode, pad, C, H, W, "float32", "paper")
            except FcfsError as e:
                assert e.name == "FCFS_E_PAD" and pad == "reflect"
                continue
            y = pl.run(x.to(DEV))
            ref = oracle.staged(x.numpy(), 5, 3, mode, pad)
            compare(y, ref, "float32", mode, float(x.max() - x.min()) or 1.0, f"{N}x{C}x{H}x{W} {mode} {pad}")


def test_empty_batch_and_errors():
    pl = Plan(3, 2, "bilinear", "replicate", 2, 16, 16, "float32")
    x = torch.empty((0, 2, 16, 16), device=DEV)
    assert pl.run(x).shape == (0, 2, 24, 24)
    from paper_2203_10670_b200 import _lib
    import ctypes
    buf = torch.zeros(2 * 16 * 16 * 4, device=DEV)
    st = _lib.lib.fcfs_run(pl.handle, ctypes.c_void_p(buf.data_ptr()), ctypes.c_void_p(buf.data_ptr() + 64), 1, None)
    assert _lib.STATUS[st] == "FCFS_E_ARG"  # overlapping in/out
    st = _lib.lib.fcfs_run(pl.handle, None, ctypes.c_void_p(buf.data_ptr()), 1, None)
    assert _lib.STATUS[st] == "FCFS_E_ARG"


def test_run_host_end_to_end():
    cfg = synth.CONFIGS["C3"]
    x = synth.make_input(cfg, 0, 2).pin_memory()
    pl = Plan(cfg.p, cfg.q, cfg.mode, cfg.pad, cfg.C, cfg.H, cfg.W, cfg.dtype, "floor")
    out = torch.empty((2, cfg.C, 213, 213), dtype=x.dtype).pin_memory()
    din = torch.empty_like(x, device=DEV)
    dout = torch.empty(out.shape, dtype=x.dtype, device=DEV)
    pl.run_host(x, out, din, dout)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), pl.run(x.to(DEV)).cpu().view(torch.int16))
    # every buffer is validated before anything is enqueued
    with pytest.raises(TypeError):
        pl.run_host(x.float(), out, din, dout)
    with pytest.raises(ValueError):
        pl.run_host(x, out[:, :, :212], din, dout)
    with pytest.raises(ValueError):
        pl.run_host(x, out, din, dout[:1])
    with pytest.raises(TypeError):
        pl.run_host(x, out, din.cpu(), dout)
    with pytest.raises(TypeError):
        pl.run_host(x.to(DEV), out, din, dout)


def test_run_batch_matches_single_runs():
    """A multi-scale pyramid of one batch in one fcfs_run_batch call (nearest
    levels share a launch) equals the individual runs bit for bit."""
    x = _rand_input(21, (2, 3, 96, 160), "float32").to(DEV)
    specs = [(2, 3, "nearest"), (3, 4, "nearest"), (1, 2, "nearest"), (5, 3, "bicubic"), (3, 5, "nearest"),
             (7, 5, "bilinear")]
    plans = [Plan(p, q, m, "replicate", 3, 96, 160, "float32", "floor") for p, q, m in specs]
    outs = [torch.empty((2, 3, pl.Ho, pl.Wo), device=DEV) for pl in plans]
    fc.run_batch([(pl, x, o) for pl, o in zip(plans, outs)])
    torch.cuda.synchronize()
    for pl, o in zip(plans, outs):
        assert torch.equal(o, pl.run(x))
    # overlapping jobs are refused before anything runs
    with pytest.raises(FcfsError) as e:
        fc.run_batch([(plans[0], x, outs[0]), (plans[0], x, outs[0])])
    assert e.value.name == "FCFS_E_ARG"


def test_streams_and_concurrency():
    cfg = synth.CONFIGS["C4b"]
    x = synth.make_input(cfg, 0, 2).to(DEV)
    pl = Plan(cfg.p, cfg.q, cfg.mode, cfg.pad, cfg.C, cfg.H, cfg.W, cfg.dtype, "floor")
    ref = pl.run(x)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        a = pl.run(x)
    with torch.cuda.stream(s2):
        b = pl.run(x)
    torch.cuda.synchronize()
    assert torch.equal(a, ref) and torch.equal(b, ref)


@pytest.mark.parametrize("mode", ["bilinear", "bicubic"])
@pytest.mark.parametrize("dtype", DTYPES)
def test_tiled_kernel_paper_factors(mode, dtype):
    """Factors without a fused variant (the paper's §6 factor 27/11,
    PAPER.md:289-300, strong down-scaling 2/13 -- the direct-tap mode -- and
    others) run the tiled kernel; 2/11 (the paper's other §6 factor) has a fused
    variant.  Many tiles with ragged edges, bitwise equal to the reference kernel
    and within the bar of the oracle."""
    for i, (p, q) in enumerate([(2, 13), (27, 11), (9, 7), (1, 6), (11, 4), (13, 10), (2, 11)]):
        pad = ["zero", "replicate", "reflect"][i % 3]
        x = _rand_input(2000 + i, (1, 2, 157, 229), dtype)
        pl = Plan(p, q, mode, pad, 2, 157, 229, dtype, "floor")
        assert pl.kernel == ("fused_separable" if (p, q) == (2, 11) else "tiled"), (p, q, pl.kernel)
        y = pl.run(x.to(DEV))
        yr = Plan(p, q, mode, pad, 2, 157, 229, dtype, "floor", force_reference=True).run(x.to(DEV))
        assert torch.equal(y.cpu().view(torch.uint8), yr.cpu().view(torch.uint8)), f"{p}/{q} {mode} {pad} kernels"
        xr = oracle_input(x)
        ref = oracle.staged(xr, p, q, mode, pad, floor_extent=True)
        compare(y, ref, dtype, mode, float(xr.max() - xr.min()), f"tiled {p}/{q} {mode} {pad} {dtype}",
                x_absmax=float(np.abs(xr).max()))


@pytest.mark.parametrize("pad", ["zero", "replicate", "reflect"])
def test_unaligned_rows_fused(pad):
    """Rows whose pitch (or start) is not 16-B aligned: the fused kernel lands
    each row's aligned superset and reads it in place at a per-row element shift
    (2D) or realigns it (3D).  Every output against the oracle and, bitwise,
    against the reference kernel; several planes so the shift varies by row and
    plane; odd element offsets for the 16-bit types."""
    for (p, q), dtype, (H, W), off in itertools.product([(5, 3), (3, 5), (7, 4), (2, 1)], DTYPES,
                                                         [(23, 37), (9, 101), (30, 250)], (0, 1)):
        N, C = 2, 3
        n = N * C * H * W
        base = _rand_input(77 + W + off, (n + off,), dtype).to(DEV)
        x = base[off:].view(N, C, H, W)
        pl = Plan(p, q, "bicubic", pad, C, H, W, dtype, "floor")
        if pad == "reflect" and min(H, W) < 3:
            continue
        y = pl.run(x)
        if off == 0:
            assert pl.launch_info(N)["kernel"] == "fused_separable", (p, q, dtype, W)
        xr = oracle_input(x.cpu())
        ref = oracle.staged(xr, p, q, "bicubic", pad, floor_extent=True)
        compare(y, ref, dtype, "bicubic", float(xr.max() - xr.min()), f"unaligned {p}/{q} {pad} {dtype} {H}x{W}+{off}",
                x_absmax=float(np.abs(xr).max()))
        yr = Plan(p, q, "bicubic", pad, C, H, W, dtype, "floor", force_reference=True).run(x)
        assert torch.equal(y.view(torch.uint8), yr.view(torch.uint8)), (p, q, pad, dtype, W, off)


def test_unaligned_strips_equal_whole_image():
    """Row strips of an image whose rows are not 16-B aligned (the fused kernel's
    in-place shifted reads with a row window) reproduce the single launch."""
    for (p, q, mode, pad, dtype) in [(5, 3, "bicubic", "reflect", "bfloat16"), (3, 5, "bicubic", "replicate", "float16"),
                                     (7, 4, "bilinear", "zero", "float32")]:
        H, W = 331, 641
        x = _rand_input(19, (2, 2, H, W), dtype).to(DEV)
        pl = Plan(p, q, mode, pad, 2, H, W, dtype, "floor")
        assert pl.launch_info(2)["kernel"] == "fused_separable"
        whole = pl.run(x)
        parts = []
        for g in range(3):
            own0, own1 = g * H // 3, (g + 1) * H // 3
            o0, o1, n0, n1 = pl.strip_rows(own0, own1)
            parts.append(pl.run_rows(x[:, :, n0:n1].contiguous(), n0, o0, o1 - o0))
        assert torch.equal(torch.cat(parts, dim=2).view(torch.uint8), whole.view(torch.uint8)), (p, q, dtype)
