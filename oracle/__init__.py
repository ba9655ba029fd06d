"""CPU oracle for FCFS (arXiv 2203.10670) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
and ``--impl reference`` legs may import this package.  The product package
``paper_2203_10670_b200`` never imports it, and this package imports nothing
from the product: the two share no code (inputs come from ``synth``).

The arithmetic lives in ``fcfs_oracle.c`` (plain C, double precision,
``-ffp-contract=off``); this module only builds it, marshals numpy arrays and
rounds the double result to the output dtype with library casts:
double -> float32 (IEEE round-to-nearest-even, numpy) -> float16 (numpy,
RNE) or bfloat16 (torch CPU ``.to(torch.bfloat16)``, RNE).  That rounding is
what BASELINE.json's "oracle's fp32 result rounded to the output dtype" means.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fcfs_oracle.c")
_LIB = os.path.join(_HERE, "libfcfs_oracle.so")

MODES = {"nearest": 0, "bilinear": 1, "bicubic": 2}
PADS = {"zero": 0, "replicate": 1, "reflect": 2}
ERRORS = {-1: "argument", -2: "padding", -3: "shape", -4: "no memory", -5: "row window"}

_lock = threading.Lock()
_lib = None


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle {what}: error {code} ({ERRORS.get(code, '?')})")
        self.code = code


def build(force: bool = False) -> str:
    """Compile fcfs_oracle.c into libfcfs_oracle.so (gcc, OpenMP, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
               "-fno-fast-math", "-Wall", "-o", tmp, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            i64, i32, dp, vp = ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p
            lib.fcfs_oracle_cubic_weight.restype = ctypes.c_double
            lib.fcfs_oracle_cubic_weight.argtypes = [ctypes.c_double]
            lib.fcfs_oracle_phase_taps.argtypes = [i32, i32, i32, i32, ctypes.POINTER(i32), dp]
            lib.fcfs_oracle_kernel2d.argtypes = [i32, i32, i32, i32, i32, ctypes.POINTER(i32),
                                                 ctypes.POINTER(i32), dp]
            lib.fcfs_oracle_pad1d.argtypes = [dp, i64, i64, i64, i32, dp]
            lib.fcfs_oracle_strided_conv1d.argtypes = [dp, i64, dp, i32, i32, i32, dp, ctypes.POINTER(i64)]
            lib.fcfs_oracle_pixelshuffle1d.argtypes = [dp, i32, i64, dp]
            lib.fcfs_oracle_pixelshuffle2d.argtypes = [dp, i32, i32, i64, i64, dp]
            lib.fcfs_oracle_output_extent.argtypes = [i64, i32, i32, i32, ctypes.POINTER(i64)]
            run_args = [vp, i32, i64, i64, i64, i64, i64, i32, i32, i32, i32, i32, i32, i64, i64, dp, i32]
            lib.fcfs_oracle_staged.argtypes = run_args
            lib.fcfs_oracle_direct_rows.argtypes = run_args
            lib.fcfs_oracle_direct_points.argtypes = [vp, i32, i64, i64, i64, i64, i64, i32, i32, i32,
                                                      i32, i32, i32, ctypes.POINTER(i64), i64, dp, i32]
            nd_args = [vp, i32, i64, i32, ctypes.POINTER(i64), ctypes.POINTER(i32), ctypes.POINTER(i32), i32, i32,
                       i32, dp, i32]
            lib.fcfs_oracle_staged_nd.argtypes = nd_args
            lib.fcfs_oracle_direct_nd.argtypes = nd_args
            lib.fcfs_oracle_adjoint_nd.argtypes = [dp, i64, i32, ctypes.POINTER(i64), ctypes.POINTER(i32),
                                                   ctypes.POINTER(i32), i32, i32, i32, dp, i32]
            lib.fcfs_oracle_output_dims_nd.argtypes = [i32, ctypes.POINTER(i64), ctypes.POINTER(i32),
                                                       ctypes.POINTER(i32), i32, ctypes.POINTER(i64)]
            lib.fcfs_oracle_weight_grad.argtypes = [vp, i32, i64, i64, i64, dp, i32, i32, i32, i32, i32, i32, dp, dp]
            lib.fcfs_oracle_weight_grad_2d.argtypes = [vp, i32, i64, i64, i64, dp, i32, i32, i32, i32, i32, i32, i32,
                                                       dp, dp]
            _lib = lib
    return _lib


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _chk(rc: int, what: str):
    if rc != 0:
        raise OracleError(rc, what)


# ---------------------------------------------------------------- primitives
def cubic_weight(delta: float) -> float:
    return _load().fcfs_oracle_cubic_weight(float(delta))


def phase_taps(mode: str, p: int, q: int, j: int):
    """(first tap offset relative to q*i, weights) of phase j (§3.1.1, §5.2)."""
    w = np.zeros(4)
    first = ctypes.c_int()
    n = _load().fcfs_oracle_phase_taps(MODES[mode], p, q, j, ctypes.byref(first), _dptr(w))
    _chk(n if n < 0 else 0, "phase_taps")
    return first.value, w[:n].copy()


def kernel2d(mode: str, p: int, q: int, jy: int, jx: int):
    """(T, lo, K) -- the T x T conv kernel of output channel (jy, jx) (§4.2)."""
    K = np.zeros(4 * 64 * 4 * 64)
    T, lo = ctypes.c_int(), ctypes.c_int()
    _chk(_load().fcfs_oracle_kernel2d(MODES[mode], p, q, jy, jx, ctypes.byref(T), ctypes.byref(lo), _dptr(K)),
         "kernel2d")
    t = T.value
    return t, lo.value, K[: t * t].reshape(t, t).copy()


def pad1d(x, left: int, right: int, pad: str) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros(x.size + left + right)
    _chk(_load().fcfs_oracle_pad1d(_dptr(x), x.size, left, right, PADS[pad], _dptr(out)), "pad1d")
    return out


def strided_conv1d(x, kernels, stride: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    k = np.ascontiguousarray(kernels, dtype=np.float64)
    C, T = k.shape
    out = np.zeros(C * max(1, (x.size - T) // stride + 1))
    n = ctypes.c_int64()
    _chk(_load().fcfs_oracle_strided_conv1d(_dptr(x), x.size, _dptr(k), C, T, stride, _dptr(out),
                                            ctypes.byref(n)), "strided_conv1d")
    return out[: C * n.value].reshape(C, n.value)


def pixelshuffle1d(h) -> np.ndarray:
    h = np.ascontiguousarray(h, dtype=np.float64)
    r, n = h.shape
    out = np.zeros(r * n)
    _load().fcfs_oracle_pixelshuffle1d(_dptr(h), r, n, _dptr(out))
    return out


def pixelshuffle2d(h, r1: int, r2: int) -> np.ndarray:
    h = np.ascontiguousarray(h, dtype=np.float64)
    c, n1, n2 = h.shape
    assert c == r1 * r2
    out = np.zeros(r1 * n1 * r2 * n2)
    _load().fcfs_oracle_pixelshuffle2d(_dptr(h), r1, r2, n1, n2, _dptr(out))
    return out.reshape(r1 * n1, r2 * n2)


def output_extent(n: int, p: int, q: int, floor_extent: bool) -> int:
    out = ctypes.c_int64()
    _chk(_load().fcfs_oracle_output_extent(n, p, q, int(floor_extent), ctypes.byref(out)), "output_extent")
    return out.value


def output_shape(H: int, W: int, p: int, q: int, floor_extent: bool, is1d: bool = False):
    return (H if is1d else output_extent(H, p, q, floor_extent)), output_extent(W, p, q, floor_extent)


# ---------------------------------------------------------------- pipeline
def _as_input(x: np.ndarray):
    if x.dtype == np.float32:
        return np.ascontiguousarray(x), 1
    return np.ascontiguousarray(x, dtype=np.float64), 0


def _run(fn, x, p, q, mode, pad, floor_extent, is1d, rows, H, row0, nthreads):
    xa, kind = _as_input(x)
    planes = int(np.prod(xa.shape[:-2])) if xa.ndim > 2 else 1
    nrows, W = xa.shape[-2], xa.shape[-1]
    Hg = nrows if H is None else H
    Ho, Wo = output_shape(Hg, W, p, q, floor_extent, is1d)
    r0, r1 = (0, Ho) if rows is None else rows
    out = np.empty((planes, r1 - r0, Wo))
    rc = fn(xa.ctypes.data, kind, planes, Hg, W, row0, nrows, p, q, MODES[mode], PADS[pad],
            int(floor_extent), int(is1d), r0, r1, _dptr(out), nthreads)
    _chk(rc, fn.__name__)
    return out.reshape(tuple(xa.shape[:-2]) + (r1 - r0, Wo))


def staged(x, p, q, mode="bilinear", pad="replicate", floor_extent=False, is1d=False, rows=None,
           H=None, row0=0, nthreads=0) -> np.ndarray:
    """The paper's layer (pad -> strided conv -> pixelshuffle -> crop) in double.

    x: (..., nrows, W) float32 or float64 holding global rows [row0, row0+nrows)
    of an H-row image (H defaults to nrows).  rows=(r0, r1) selects output rows.
    """
    return _run(_load().fcfs_oracle_staged, x, p, q, mode, pad, floor_extent, is1d, rows, H, row0, nthreads)


def direct(x, p, q, mode="bilinear", pad="replicate", floor_extent=False, is1d=False, rows=None,
           H=None, row0=0, nthreads=0) -> np.ndarray:
    """Per-output direct evaluation of the interpolation formula (independent code)."""
    return _run(_load().fcfs_oracle_direct_rows, x, p, q, mode, pad, floor_extent, is1d, rows, H, row0,
                nthreads)


def direct_points(x, pts, p, q, mode="bilinear", pad="replicate", floor_extent=False, is1d=False,
                  H=None, row0=0, nthreads=0) -> np.ndarray:
    """Direct evaluation at sampled outputs pts[i] = (plane, my, mx)."""
    xa, kind = _as_input(x)
    planes = int(np.prod(xa.shape[:-2])) if xa.ndim > 2 else 1
    nrows, W = xa.shape[-2], xa.shape[-1]
    Hg = nrows if H is None else H
    pts = np.ascontiguousarray(pts, dtype=np.int64).reshape(-1, 3)
    out = np.empty(pts.shape[0])
    rc = _load().fcfs_oracle_direct_points(
        xa.ctypes.data, kind, planes, Hg, W, row0, nrows, p, q, MODES[mode], PADS[pad], int(floor_extent),
        int(is1d), pts.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), pts.shape[0], _dptr(out), nthreads)
    _chk(rc, "direct_points")
    return out


# ---------------------------------------------------------------- ND, per-dimension factors (§4.2)
def _nd_params(p, q, R):
    p = [int(v) for v in (p if hasattr(p, "__len__") else [p] * R)]
    q = [int(v) for v in (q if hasattr(q, "__len__") else [q] * R)]
    if len(p) != R or len(q) != R:
        raise ValueError("one factor per spatial dimension")
    return (ctypes.c_int * R)(*p), (ctypes.c_int * R)(*q)


def output_dims_nd(dims, p, q, floor_extent=False):
    R = len(dims)
    pp, qq = _nd_params(p, q, R)
    d = (ctypes.c_int64 * R)(*dims)
    out = (ctypes.c_int64 * R)()
    _chk(_load().fcfs_oracle_output_dims_nd(R, d, pp, qq, int(floor_extent), out), "output_dims_nd")
    return tuple(out)


def _run_nd(fn, x, p, q, R, mode, pad, floor_extent, nthreads):
    xa, kind = _as_input(x)
    if xa.ndim < R:
        raise ValueError("input has fewer dimensions than the rank")
    dims = xa.shape[xa.ndim - R:]
    planes = int(np.prod(xa.shape[: xa.ndim - R])) if xa.ndim > R else 1
    pp, qq = _nd_params(p, q, R)
    odims = output_dims_nd(dims, p, q, floor_extent)
    out = np.empty((planes,) + odims)
    rc = fn(xa.ctypes.data, kind, planes, R, (ctypes.c_int64 * R)(*dims), pp, qq, MODES[mode], PADS[pad],
            int(floor_extent), _dptr(out), nthreads)
    _chk(rc, fn.__name__)
    return out.reshape(tuple(xa.shape[: xa.ndim - R]) + odims)


def staged_nd(x, p, q, mode="bilinear", pad="replicate", floor_extent=False, rank=None, nthreads=0):
    """ND FCFS with per-dimension factors p[d]/q[d] (§4.2): pad -> conv with
    prod p_d channels and stride q_d -> ND pixelshuffle (§4.1) -> crop, over the
    last `rank` (= len(p)) axes of x, in double."""
    R = rank if rank is not None else (len(p) if hasattr(p, "__len__") else 2)
    return _run_nd(_load().fcfs_oracle_staged_nd, x, p, q, R, mode, pad, floor_extent, nthreads)


def direct_nd(x, p, q, mode="bilinear", pad="replicate", floor_extent=False, rank=None, nthreads=0):
    """Per-output direct evaluation of the ND interpolation formula (independent code)."""
    R = rank if rank is not None else (len(p) if hasattr(p, "__len__") else 2)
    return _run_nd(_load().fcfs_oracle_direct_nd, x, p, q, R, mode, pad, floor_extent, nthreads)


def adjoint_nd(g, dims, p, q, mode="bilinear", pad="replicate", floor_extent=False, nthreads=0):
    """A^T g for the ND layer A of (dims, p, q, mode, pad): the input gradient
    (backward pass).  g: (..., *odims); returns (..., *dims), double."""
    R = len(dims)
    pp, qq = _nd_params(p, q, R)
    odims = output_dims_nd(dims, p, q, floor_extent)
    ga = np.ascontiguousarray(g, dtype=np.float64)
    if tuple(ga.shape[ga.ndim - R:]) != tuple(odims):
        raise ValueError(f"gradient shape {ga.shape} does not end with the output dims {odims}")
    lead = ga.shape[: ga.ndim - R]
    planes = int(np.prod(lead)) if lead else 1
    out = np.empty((planes,) + tuple(dims))
    rc = _load().fcfs_oracle_adjoint_nd(_dptr(ga), planes, R, (ctypes.c_int64 * R)(*dims), pp, qq, MODES[mode],
                                        PADS[pad], int(floor_extent), _dptr(out), nthreads)
    _chk(rc, "adjoint_nd")
    return out.reshape(tuple(lead) + tuple(dims))


def weight_grad(x, g, p, q, mode="bilinear", pad="replicate", floor_extent=False, is1d=False):
    """Gradient of sum(y * g) with respect to the layer's learnable weights
    (reading Z22: each output channel's own taps), summed over all planes.

    x: (..., H, W) float32 or float64; g: (..., Ho, Wo) (the layer output's shape).
    Returns (grad, abs_sum), both double of shape (py, px, nty, ntx) -- 2D: (p, p,
    taps, taps); 1D flag: (1, p, 1, taps) -- abs_sum the same sums of |g| |x|.
    """
    xa, kind = _as_input(x)
    H, W = xa.shape[-2], xa.shape[-1]
    planes = int(np.prod(xa.shape[:-2])) if xa.ndim > 2 else 1
    Ho, Wo = output_shape(H, W, p, q, floor_extent, is1d)
    ga = np.ascontiguousarray(g, dtype=np.float64)
    if ga.size != planes * Ho * Wo:
        raise ValueError(f"gradient of {ga.size} elements, expected {planes} x {Ho} x {Wo}")
    from math import gcd
    pr = p // gcd(p, q)
    nt = {"nearest": 1, "bilinear": 2, "bicubic": 4}[mode]
    shape = (1, pr, 1, nt) if is1d else (pr, pr, nt, nt)
    out, ab = np.zeros(shape), np.zeros(shape)
    rc = _load().fcfs_oracle_weight_grad(xa.ctypes.data, kind, planes, H, W, _dptr(ga), p, q, MODES[mode],
                                         PADS[pad], int(floor_extent), int(is1d), _dptr(out), _dptr(ab))
    _chk(rc, "weight_grad")
    return out, ab


def weight_grad_2d(x, g, p, q, mode="bilinear", pad="replicate", floor_extent=False):
    """weight_grad for a 2D layer with a factor per dimension: p = (py, px), q = (qy, qx).
    Returns (grad, abs_sum) of shape (py, px, taps, taps) (reduced factors)."""
    from math import gcd
    xa, kind = _as_input(x)
    H, W = xa.shape[-2], xa.shape[-1]
    planes = int(np.prod(xa.shape[:-2])) if xa.ndim > 2 else 1
    (py, px), (qy, qx) = p, q
    Ho, Wo = output_extent(H, py, qy, floor_extent), output_extent(W, px, qx, floor_extent)
    ga = np.ascontiguousarray(g, dtype=np.float64)
    if ga.size != planes * Ho * Wo:
        raise ValueError(f"gradient of {ga.size} elements, expected {planes} x {Ho} x {Wo}")
    nt = {"nearest": 1, "bilinear": 2, "bicubic": 4}[mode]
    shape = (py // gcd(py, qy), px // gcd(px, qx), nt, nt)
    out, ab = np.zeros(shape), np.zeros(shape)
    rc = _load().fcfs_oracle_weight_grad_2d(xa.ctypes.data, kind, planes, H, W, _dptr(ga), py, qy, px, qx,
                                            MODES[mode], PADS[pad], int(floor_extent), _dptr(out), _dptr(ab))
    _chk(rc, "weight_grad_2d")
    return out, ab


# ---------------------------------------------------------------- rounding
def round_to(y: np.ndarray, dtype: str):
    """double -> float32 (RNE) -> dtype (RNE).  Returns a torch CPU tensor for
    bfloat16, numpy otherwise ("the oracle's fp32 result rounded to the output
    dtype", BASELINE.json north_star)."""
    f32 = np.asarray(y, dtype=np.float64).astype(np.float32)
    if dtype in ("float32", "f32"):
        return f32
    if dtype in ("float16", "f16"):
        return f32.astype(np.float16)
    if dtype in ("bfloat16", "bf16"):
        import torch
        return torch.from_numpy(f32).to(torch.bfloat16)
    raise ValueError(dtype)
