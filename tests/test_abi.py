"""Host-side checks of libfcfs.so (no GPU needed): it loads, exports every
symbol include/fcfs.h declares, and its host logic (validation, extents, phase
table, strip ownership, byte accounting, status codes) is right."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fcfs.h")


@pytest.fixture(scope="module")
def fc():
    import paper_2203_10670_b200 as fc
    return fc


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fcfs_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(fc):
    names = declared_functions()
    assert "fcfs_plan" in names and "fcfs_run" in names and "fcfs_destroy" in names and len(names) >= 13
    lib = ctypes.CDLL(fc.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    nm = subprocess.run(["nm", "-D", "--defined-only", fc.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (fcfs_\w+)", nm))
    assert set(names) <= exported
    # the binding declares exactly the header's functions
    from paper_2203_10670_b200 import _lib
    assert set(_lib.SIGNATURES) == set(names)


def test_library_is_sm100a(fc):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", fc.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_or_torch_in_product_path():
    pkg = os.path.join(ROOT, "paper_2203_10670_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "fcfs_oracle" not in src, f
    # the oracle includes nothing from the product
    osrc = open(os.path.join(ROOT, "oracle", "fcfs_oracle.c")).read()
    assert "fcfs.h" not in osrc and "fcfs_internal" not in osrc


@pytest.mark.parametrize("p,q,H,W,floor,out", [(3, 2, 5, 5, False, (9, 9)), (3, 2, 48, 64, True, (72, 96)),
                                                (5, 3, 128, 128, True, (213, 213)), (5, 3, 128, 128, False, (215, 215)),
                                                (2, 11, 1024, 1024, False, (188, 188)), (6, 4, 5, 5, False, (9, 9)),
                                                (7, 5, 2160, 3840, True, (3024, 5376)),
                                                (4, 7, 2160, 3840, True, (1234, 2194)),
                                                (3, 5, 32768, 32768, True, (19660, 19660))])
def test_output_shapes(fc, p, q, H, W, floor, out):
    pl = fc.Plan(p, q, "bilinear", "replicate", 1, H, W, "float32", "floor" if floor else "paper")
    assert pl.output_shape() == out
    assert pl.output_shape() == oracle.output_shape(H, W, p, q, floor)


def test_errors(fc):
    from paper_2203_10670_b200._lib import FcfsError
    cases = [((0, 1, "bilinear", "zero", 1, 4, 4), "FCFS_E_ARG"), ((65, 1, "bilinear", "zero", 1, 4, 4), "FCFS_E_ARG"),
             ((1, 1, "bilinear", "zero", 0, 4, 4), "FCFS_E_ARG"), ((1, 1, "bilinear", "zero", 1, 0, 4), "FCFS_E_ARG"),
             ((5, 3, "bicubic", "reflect", 1, 1, 8), "FCFS_E_PAD"), ((3, 2, "bilinear", "reflect", 1, 8, 1), "FCFS_E_PAD")]
    for args, name in cases:
        with pytest.raises(FcfsError) as e:
            fc.Plan(*args)
        assert e.value.name == name, args
    with pytest.raises(FcfsError) as e:
        fc.Plan(2, 11, "bilinear", "replicate", 1, 5, 5, "float32", "floor")
    assert e.value.name == "FCFS_E_SHAPE"
    # reducible factors beyond 64 are fine once reduced
    assert fc.Plan(128, 64, "nearest", "zero", 1, 4, 4).p == 2
    with pytest.raises(FcfsError):
        fc.Plan(65, 64, "nearest", "zero", 1, 4, 4)


def test_unknown_enum_and_flags():
    from paper_2203_10670_b200 import _lib
    h = ctypes.c_void_p()
    assert _lib.lib.fcfs_plan_ex(3, 2, 7, 0, 1, 4, 4, 0, 0, ctypes.byref(h)) == 1
    assert _lib.lib.fcfs_plan_ex(3, 2, 0, 9, 1, 4, 4, 0, 0, ctypes.byref(h)) == 1
    assert _lib.lib.fcfs_plan_ex(3, 2, 0, 0, 1, 4, 4, 5, 0, ctypes.byref(h)) == 1
    assert _lib.lib.fcfs_plan_ex(3, 2, 0, 0, 1, 4, 4, 0, 1 << 20, ctypes.byref(h)) == 1
    assert _lib.lib.fcfs_plan_ex(3, 2, 0, 0, 1, 4, 4, 0, 0, None) == 1
    assert _lib.lib.fcfs_status_str(6).decode() == "CUDA error"
    assert _lib.lib.fcfs_version() == 5


def test_run_without_device_is_refused(fc):
    import torch
    if torch.cuda.is_available():
        pytest.skip("host without GPU only")
    from paper_2203_10670_b200 import _lib
    pl = fc.Plan(3, 2, "bilinear", "replicate", 1, 8, 8)
    assert pl.info.device == -1
    st = _lib.lib.fcfs_run(pl.handle, ctypes.c_void_p(0x1000), ctypes.c_void_p(0x100000), 1, None)
    assert _lib.STATUS[st] == "FCFS_E_DEVICE"


@pytest.mark.parametrize("mode", ["nearest", "bilinear", "bicubic"])
@pytest.mark.parametrize("p,q", [(3, 2), (5, 3), (7, 5), (4, 7), (3, 5), (27, 11), (1, 1)])
def test_phase_table_matches_oracle_weights(fc, mode, p, q):
    pl = fc.Plan(p, q, mode, "replicate", 1, 64, 64)
    w, base = pl.phase_table()
    for j in range(p):
        first, ow = oracle.phase_taps(mode, p, q, j)
        assert base[j] == (j * q) // p
        assert first - base[j] == pl.info.lo
        # fp32 rounding of the exact weight (the oracle keeps double)
        np.testing.assert_array_equal(np.float32(ow), np.float32(w[j][: len(ow)]))
        assert all(v == 0 for v in w[j][len(ow):])


def test_kernel_selection(fc):
    assert fc.Plan(5, 3, "bicubic", "reflect", 1, 128, 128, "bfloat16").kernel == "fused_separable"
    assert fc.Plan(2, 3, "nearest", "zero", 1, 512, 512).kernel == "nearest_gather"
    assert fc.Plan(27, 11, "bicubic", "replicate", 1, 64, 64).kernel == "tiled"  # no fused variant
    assert fc.Plan(3, 2, "bilinear", "replicate", 1, 64, 101).kernel == "fused_separable"  # unaligned pitch: software row copies
    # 1D rows run the fused kernel with a 1/1 row factor (the "width-only" variants)
    assert fc.Plan(3, 2, "bilinear", "replicate", 1, 64, 64, is1d=True).kernel == "fused_separable"
    assert fc.Plan(3, 2, "bilinear", "replicate", 1, 64, 64, force_reference=True).kernel == "reference"
    # per-dimension factors (§4.2)
    assert fc.Plan.nd((1, 3), (1, 4), "bicubic", "reflect", 3, (64, 64), "float16").kernel == "fused_separable"
    assert fc.Plan.nd((5, 1), (3, 1), "bilinear", "zero", 3, (64, 64), "bfloat16").kernel == "fused_separable"
    assert fc.Plan.nd((5, 3), (3, 4), "bilinear", "zero", 3, (64, 64)).kernel == "tiled"  # no variant
    assert fc.Plan.nd((2, 3, 5), (1, 2, 3), "nearest", "zero", 1, (8, 16, 16)).kernel == "nearest_gather"
    assert fc.Plan.nd((2, 3, 3), (1, 2, 2), "bicubic", "zero", 1, (8, 16, 16)).kernel == "fused_separable"
    assert fc.Plan.nd((7, 5, 5), (3, 3, 3), "bilinear", "zero", 1, (8, 16, 16)).kernel == "fused_separable"
    assert fc.Plan.nd((2, 3, 5), (1, 2, 3), "bicubic", "zero", 1, (8, 16, 16)).kernel == "reference"  # y != x
    assert fc.Plan.nd((17, 3, 3), (5, 2, 2), "bicubic", "zero", 1, (8, 16, 16)).kernel == "reference"  # pz > 16
    assert fc.Plan.nd((1, 3, 3), (1, 2, 2), "bicubic", "zero", 1, (8, 16, 16)).kernel == "fused_separable"
    assert fc.Plan.nd([3], [2], "bilinear", "zero", 2, (64,)).kernel == "fused_separable"


def test_nd_plan_shapes_and_tables(fc):
    """Per-dimension extents, info fields and phase tables against the oracle."""
    import oracle
    for dims, p, q, mode in [((9, 17, 32), (3, 2, 5), (2, 3, 3), "bicubic"), ((40, 24), (5, 1), (3, 4), "bilinear"),
                             ((101,), (2,), (3,), "nearest")]:
        for ext in ("paper", "floor"):
            pl = fc.Plan.nd(p, q, mode, "replicate", 2, dims, "float32", ext)
            R = len(dims)
            assert pl.rank == R and pl.dims == dims
            assert pl.odims == oracle.output_dims_nd(dims, p, q, ext == "floor")
            assert pl.factors == tuple(zip(p, q))
            for d in range(R):
                w = (ctypes.c_float * (4 * p[d]))()
                b = (ctypes.c_int * p[d])()
                assert fc._lib.lib.fcfs_phase_table_dim(pl.handle, d, w, b) == 0
                for j in range(p[d]):
                    first, ow = oracle.phase_taps(mode, p[d], q[d], j)
                    assert b[j] == (j * q[d]) // p[d]
                    np.testing.assert_array_equal(np.float32(ow), np.float32(list(w)[4 * j: 4 * j + len(ow)]))
            od = (ctypes.c_int64 * R)()
            assert fc._lib.lib.fcfs_output_dims(pl.handle, od) == 0 and tuple(od) == pl.odims
            assert fc._lib.lib.fcfs_phase_table_dim(pl.handle, R, w, b) == 1  # FCFS_E_ARG
    # rank outside 1..3, 1D flag with the ND form, reflect that cannot reach (D = 2, bicubic up)
    h = ctypes.c_void_p()
    one = (ctypes.c_int * 4)(1, 1, 1, 1)
    dims4 = (ctypes.c_int64 * 4)(2, 2, 2, 2)
    assert fc._lib.lib.fcfs_plan_nd(4, one, one, 1, 0, 1, dims4, 0, 0, ctypes.byref(h)) == 1
    assert fc._lib.lib.fcfs_plan_nd(2, one, one, 1, 0, 1, dims4, 0, 1, ctypes.byref(h)) == 1
    with pytest.raises(fc.FcfsError):
        fc.Plan.nd((5, 1, 1), (2, 1, 1), "bicubic", "reflect", 1, (2, 8, 8))


@pytest.mark.parametrize("name", ["C1a", "C1b", "C2a", "C2b", "C3", "C4a", "C4b", "C5"])
def test_launch_geometry(fc, name):
    """The planner's launch geometry for every config: fits the shared-memory
    budget (2 CTAs/SM), keeps at least ~85% of the consumer threads busy on the
    big configs, and tiles the output exactly."""
    import synth
    c = synth.CONFIGS[name]
    pl = fc.Plan(c.p, c.q, c.mode, c.pad, c.C, c.H, c.W, c.dtype, "floor", c.is1d)
    info = pl.launch_info(c.N)
    if info["kernel"] == "fused_plane":
        # batches of small planes (C3): whole padded planes per TMA box, a warp per
        # band across the full output width, two CTAs per SM
        assert pl.kernel == "fused_separable"
        assert info["smem"] <= 112 * 1024 and info["BW"] <= 256 and info["BH"] <= 256
        assert info["nch"] <= 32 and info["nch"] * info["K"] * info["PX"] >= pl.Wo
        assert info["grid"] == min(c.N * c.C, 296) and info["block"] == 256
        assert info["BH"] >= (info["periods"] - 1) * info["QY"] + 1
        return
    assert info["kernel"] == pl.kernel
    if info["kernel"] != "fused_separable":
        return
    assert info["smem"] <= 113 * 1024 and info["S"] >= 2 and info["grid"] <= 296
    assert info["CPT"] * info["ntile"] >= info["nch"] and info["NS"] * info["CPT"] <= 256
    assert info["nch"] * info["K"] * info["PX"] >= pl.Wo
    assert info["PB"] * info["nbands"] >= info["periods"]
    assert info["ntasks"] == -(-info["nseg"] // info["NS"]) * info["nbands"]
    if name in ("C3", "C4a", "C4b", "C5"):
        # C5 (fp32 3/5, K = 3: 45 input columns x 5 fresh rows per thread) is
        # bound by the shared-memory budget instead: 146 threads, measured faster
        # than 253 threads at K = 1 (1012 vs 1044 us)
        assert info["busy_threads"] >= (0.55 if name == "C5" else 0.85) * 256
        assert info["ntasks"] >= 296  # every SM slot has work


def _own(p, q, H, Ho, own0, own1):
    """Brute force: outputs whose base row floor(m*q/p) lies in [own0, own1)."""
    ms = [m for m in range(Ho) if own0 <= (m * q) // p < own1 or (own1 == H and (m * q) // p >= H)]
    return (ms[0], ms[-1] + 1) if ms else None


@pytest.mark.parametrize("p,q,mode,pad,ext", [(3, 5, "bicubic", "replicate", "floor"), (5, 3, "bicubic", "reflect", "paper"),
                                              (7, 5, "bilinear", "zero", "floor"), (2, 3, "nearest", "zero", "paper"),
                                              (4, 7, "bilinear", "replicate", "paper")])
def test_strip_rows_partition_and_halo(fc, p, q, mode, pad, ext):
    H, W = 203, 16
    pl = fc.Plan(p, q, mode, pad, 1, H, W, "float32", ext)
    Ho = pl.Ho
    for G in (1, 2, 3, 7, 8):
        prev = 0
        for g in range(G):
            own0, own1 = g * H // G, (g + 1) * H // G
            o0, o1, n0, n1 = pl.strip_rows(own0, own1)
            assert o0 == prev
            prev = o1
            bf = _own(p, q, H, Ho, own0, own1)
            assert (bf is None and o0 == o1) or bf == (o0, o1)
            if o1 > o0:
                # every row a kept output's tap reads (after global padding) is inside [n0, n1)
                taps = {"nearest": [0], "bilinear": [0, 1], "bicubic": [-1, 0, 1, 2]}[mode]
                rows = set()
                for m in range(o0, o1):
                    for t in taps:
                        v = (m * q) // p + t
                        if 0 <= v < H:
                            rows.add(v)
                        elif pad == "replicate":
                            rows.add(0 if v < 0 else H - 1)
                        elif pad == "reflect":
                            rows.add(-v if v < 0 else 2 * (H - 1) - v)
                assert min(rows) == n0 and max(rows) == n1 - 1
        assert prev == Ho


def test_compulsory_bytes(fc):
    # SURVEY.md Appendix A / BASELINE.md §3 figures
    pl = fc.Plan(2, 3, "nearest", "zero", 3, 512, 512, "float32", "floor")
    assert pl.compulsory_bytes(16) == 55847616
    pl = fc.Plan(3, 4, "nearest", "zero", 3, 512, 512, "float32", "floor")
    assert pl.compulsory_bytes(16) == 66060288
    pl = fc.Plan(5, 3, "bicubic", "reflect", 64, 128, 128, "bfloat16", "floor")
    assert pl.compulsory_bytes(64) == 505880576
    pl = fc.Plan(7, 5, "bilinear", "replicate", 3, 2160, 3840, "float16", "floor")
    assert pl.compulsory_bytes(8) == 1178468352
    pl = fc.Plan(4, 7, "bilinear", "replicate", 3, 2160, 3840, "float16", "floor")
    assert pl.compulsory_bytes(8) == 527901888


def test_round2_kernel_geometry(fc):
    """Host logic of the round-2 kernels (no GPU): which kernel a run takes and
    the geometry invariants each relies on."""
    # nearest C2: the async row kernel, four CTAs per SM at most, 8 warps each
    pl = fc.Plan(2, 3, "nearest", "zero", 3, 512, 512, "float32", "floor")
    info = pl.launch_info(16)
    assert info["kernel"] == "nearest_gather" and info["variant"] == "rows_async", info
    assert info["block"] == 256 and info["grid"] <= 4 * 148
    # V2: the slice-ring plane kernel; taps + 1 slice buffers; runs of output slices
    # per volume sized for one wave; the ring and staging fit one SM
    pl = fc.Plan.nd((5, 5, 5), (3, 3, 3), "bicubic", "reflect", 8, (64, 128, 128), "bfloat16", "floor")
    info = pl.launch_info(2)
    assert info["kernel"] == "fused_plane3", info
    assert info["S"] >= info["taps"] + 1 and info["smem"] <= 227 * 1024
    assert info["ntasks"] == 2 * 8 * info["chunks"] and info["grid"] == min(info["ntasks"], 148)
    assert info["BH"] >= (info["periods"] - 1) * info["QY"] + 1 and info["BW"] <= 256
    # f32 bicubic 128^2 slices: taps + 1 buffers do not fit -> the row-pipelined 3D kernel
    pl = fc.Plan.nd((5, 5, 5), (3, 3, 3), "bicubic", "reflect", 2, (16, 128, 128), "float32", "floor")
    assert pl.launch_info(1)["kernel"] == "fused_separable"
    # A2: height-only rows -> the column-vector kernel; every (plane, band, vector) a thread
    pl = fc.Plan.nd((5, 1), (3, 1), "bicubic", "reflect", 3, (2160, 3840), "float16", "floor")
    info = pl.launch_info(8)
    assert info["kernel"] == "fused_vpass", info
    assert info["nvec"] == 3840 * 2 // 16 and info["periods"] == -(-pl.odims[0] // 5)
    assert info["band_periods"] * info["bands"] >= info["periods"]
    assert info["grid"] * 256 >= 8 * 3 * info["nvec"] * info["bands"]
    # unaligned rows (W * esize not a 16-B multiple) keep the fused kernel
    pl = fc.Plan.nd((5, 1), (3, 1), "bicubic", "reflect", 3, (64, 101), "float32", "floor")
    assert pl.launch_info(2)["kernel"] == "fused_separable"
