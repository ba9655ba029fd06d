"""Python face of the FCFS hot path: plans and scale() over torch CUDA tensors.

torch is used only for device memory and streams; every step of the path
(pad, strided polyphase conv, pixelshuffle) runs in libfcfs.so.
"""
from __future__ import annotations

import ctypes
import threading

from . import _lib
from ._lib import FLAG_1D, FLAG_EXTENT_FLOOR, FLAG_FORCE_REFERENCE, check

_TORCH_DTYPES = None


def _dtype_name(dt) -> str:
    import torch
    names = {torch.float32: "float32", torch.float16: "float16", torch.bfloat16: "bfloat16"}
    if dt not in names:
        raise TypeError(f"FCFS supports float32, float16 and bfloat16 tensors, got {dt}")
    return names[dt]


class Plan:
    """An immutable FCFS plan (fcfs_plan_ex).

    p/q: scale factor (paper r/s); mode: nearest|bilinear|bicubic;
    pad: zero|replicate|reflect; C, H, W: one image; dtype: float32|float16|
    bfloat16; extent: "paper" (p*ceil(N/q)) or "floor" (floor(N*p/q));
    is1d: scale W only.
    """

    def __init__(self, p: int, q: int, mode: str = "bilinear", pad: str = "replicate", C: int = 1, H: int = 1,
                 W: int = 1, dtype: str = "float32", extent: str = "paper", is1d: bool = False,
                 force_reference: bool = False):
        flags = (FLAG_EXTENT_FLOOR if extent == "floor" else 0) | (FLAG_1D if is1d else 0) | \
            (FLAG_FORCE_REFERENCE if force_reference else 0)
        if extent not in ("paper", "floor"):
            raise ValueError(extent)
        h = ctypes.c_void_p()
        if isinstance(p, (tuple, list)):  # per-dimension factors: the ND form (§4.2)
            if is1d:
                raise ValueError("per-dimension plans express 1D as rank 1")
            R = len(p)
            if isinstance(H, (tuple, list)):  # Plan.nd: the spatial dims, outermost first
                dims = tuple(int(v) for v in H)
            elif R == 2:
                dims = (int(H), int(W))
            elif R == 1:
                dims = (int(W),)
            else:
                raise ValueError("rank-3 plans take dims=(D, H, W) (Plan.nd)")
            if len(q) != R or len(dims) != R:
                raise ValueError("p, q and dims need one entry per spatial dimension")
            check(_lib.lib.fcfs_plan_nd(R, (ctypes.c_int * R)(*p), (ctypes.c_int * R)(*q), _lib.MODES[mode],
                                        _lib.PADS[pad], C, (ctypes.c_int64 * R)(*dims), _lib.DTYPES[dtype], flags,
                                        ctypes.byref(h)), "fcfs_plan_nd")
        else:
            check(_lib.lib.fcfs_plan_ex(p, q, _lib.MODES[mode], _lib.PADS[pad], C, H, W, _lib.DTYPES[dtype], flags,
                                        ctypes.byref(h)), "fcfs_plan_ex")
        self._h = h
        self.mode, self.pad, self.dtype, self.extent, self.is1d = mode, pad, dtype, extent, is1d
        info = _lib.PlanInfo()
        check(_lib.lib.fcfs_plan_info(h, ctypes.byref(info)), "fcfs_plan_info")
        self.info = info
        self.p, self.q = info.p, info.q
        self.C, self.H, self.W, self.Ho, self.Wo = info.C, info.H, info.W, info.Ho, info.Wo
        self.rank = info.rank
        nd = isinstance(p, (tuple, list))
        # spatial dims of the tensors run() takes: (H, W) for fcfs_plan_ex plans
        # (FCFS_FLAG_1D included), the plan's own rank for ND plans
        r = info.rank if nd else 2
        self.dims = tuple(info.dims[:r]) if nd else (info.H, info.W)
        self.odims = tuple(info.odims[:r]) if nd else (info.Ho, info.Wo)
        self.factors = tuple(zip(info.pd[:info.rank], info.qd[:info.rank]))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and getattr(_lib, "lib", None) is not None:  # (not at interpreter shutdown)
            _lib.lib.fcfs_destroy(h)
            self._h = None

    @classmethod
    def nd(cls, p, q, mode="bilinear", pad="replicate", C=1, dims=(1,), dtype="float32", extent="paper",
           force_reference=False):
        """ND plan with per-dimension factors p[d]/q[d] over spatial dims (D, H, W order)."""
        return cls(tuple(p), tuple(q), mode, pad, C, tuple(dims), 1, dtype, extent, False, force_reference)

    @property
    def handle(self):
        return self._h

    @property
    def kernel(self) -> str:
        return _lib.KERNELS[self.info.kernel]

    def output_shape(self):
        return self.Ho, self.Wo

    def phase_table(self):
        w = (ctypes.c_float * (4 * self.p))()
        b = (ctypes.c_int * self.p)()
        check(_lib.lib.fcfs_phase_table(self._h, w, b), "fcfs_phase_table")
        return [list(w[4 * j: 4 * j + 4]) for j in range(self.p)], list(b)

    def compulsory_bytes(self, N: int) -> int:
        out = ctypes.c_int64()
        check(_lib.lib.fcfs_compulsory_bytes(self._h, N, ctypes.byref(out)), "fcfs_compulsory_bytes")
        return out.value

    def strip_rows(self, own0: int, own1: int):
        """(out_row0, out_row1, need_row0, need_row1) for a strip owning input rows [own0, own1)."""
        v = [ctypes.c_int64() for _ in range(4)]
        check(_lib.lib.fcfs_strip_rows(self._h, own0, own1, *[ctypes.byref(x) for x in v]), "fcfs_strip_rows")
        return tuple(x.value for x in v)

    def launch_info(self, N: int, out_row0: int = 0, out_nrows: int | None = None) -> dict:
        """The kernel and launch geometry a run would use (host only)."""
        import json
        buf = ctypes.create_string_buffer(1024)
        n = self.Ho - out_row0 if out_nrows is None else out_nrows
        check(_lib.lib.fcfs_launch_info(self._h, N, out_row0, n, buf, 1024), "fcfs_launch_info")
        return json.loads(buf.value.decode())

    def adjoint_info(self, N: int) -> dict:
        """The launches run_adjoint would make (host only, fcfs_adjoint_info)."""
        import json
        buf = ctypes.create_string_buffer(1024)
        check(_lib.lib.fcfs_adjoint_info(self._h, N, buf, 1024), "fcfs_adjoint_info")
        return json.loads(buf.value.decode())

    def needed_rows(self, out0: int, out1: int):
        """Input rows [need0, need1) that output rows [out0, out1) read."""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        check(_lib.lib.fcfs_needed_rows(self._h, out0, out1, ctypes.byref(a), ctypes.byref(b)), "fcfs_needed_rows")
        return a.value, b.value

    # ---------------------------------------------------------------- runs
    def _stream(self, stream):
        import torch
        s = torch.cuda.current_stream() if stream is None else stream
        return ctypes.c_void_p(s.cuda_stream)

    def _check_tensor(self, t, shape, what):
        import torch
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise TypeError(f"{what} must be a CUDA tensor")
        if _dtype_name(t.dtype) != self.dtype:
            raise TypeError(f"{what} dtype {t.dtype} does not match the plan's {self.dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{what} must be contiguous")
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{what} shape {tuple(t.shape)} != {tuple(shape)}")

    def in_shape(self, N: int):
        return (N, self.C) + self.dims

    def out_shape(self, N: int):
        return (N, self.C) + self.odims

    def run(self, x, out=None, stream=None):
        """out[N, C, *odims] = FCFS(x[N, C, *dims]) on the current (or given) stream."""
        import torch
        N = x.shape[0]
        self._check_tensor(x, self.in_shape(N), "input")
        if out is None:
            out = torch.empty(self.out_shape(N), dtype=x.dtype, device=x.device)
        self._check_tensor(out, self.out_shape(N), "output")
        check(_lib.lib.fcfs_run(self._h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), N,
                                self._stream(stream)), "fcfs_run")
        return out

    def run_adjoint(self, grad_out, out=None, stream=None):
        """grad_in[N, C, *dims] = A^T grad_out[N, C, *odims] (fcfs_run_adjoint): the backward pass."""
        import torch
        N = grad_out.shape[0]
        self._check_tensor(grad_out, self.out_shape(N), "grad_out")
        if out is None:
            out = torch.empty(self.in_shape(N), dtype=grad_out.dtype, device=grad_out.device)
        self._check_tensor(out, self.in_shape(N), "grad_in")
        check(_lib.lib.fcfs_run_adjoint(self._h, ctypes.c_void_p(grad_out.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                        N, self._stream(stream)), "fcfs_run_adjoint")
        return out

    def run_rows_segments(self, windows, out_row0: int, out_nrows: int, out=None, stream=None):
        """Output rows [out_row0, out_row0+out_nrows) from up to 3 row windows
        [(tensor (N, C, nrows, W), global row0), ...] -- e.g. neighbour strips read
        in place through peer pointers (fcfs_run_rows_segments)."""
        import torch
        if not 1 <= len(windows) <= 3:
            raise ValueError("1 to 3 row windows")
        N = windows[0][0].shape[0]
        ptrs, r0s, nrs = [], [], []
        for t, r0 in windows:
            self._check_tensor(t, (N, self.C, t.shape[2], self.W), "row window")
            ptrs.append(t.data_ptr())
            r0s.append(r0)
            nrs.append(t.shape[2])
        oshape = (N, self.C, out_nrows, self.Wo)
        if out is None:
            out = torch.empty(oshape, dtype=windows[0][0].dtype, device=windows[0][0].device)
        self._check_tensor(out, oshape, "output rows")
        n = len(windows)
        check(_lib.lib.fcfs_run_rows_segments(self._h, n, (ctypes.c_void_p * n)(*ptrs), (ctypes.c_int64 * n)(*r0s),
                                              (ctypes.c_int64 * n)(*nrs), ctypes.c_void_p(out.data_ptr()), out_row0,
                                              out_nrows, N, self._stream(stream)), "fcfs_run_rows_segments")
        return out

    def weight_grad_shape(self):
        """(py, px, nty, ntx) of the learnable taps (fcfs_weight_grad_shape; reading Z22)."""
        d = (ctypes.c_int64 * 4)()
        check(_lib.lib.fcfs_weight_grad_shape(self._h, d), "fcfs_weight_grad_shape")
        return tuple(d)

    def run_weight_grad(self, x, grad_out, out=None, stream=None):
        """d(sum y * grad_out)/dW over the learnable taps, fp32 (fcfs_run_weight_grad)."""
        import torch
        N = x.shape[0]
        self._check_tensor(x, self.in_shape(N), "x")
        self._check_tensor(grad_out, self.out_shape(N), "grad_out")
        if grad_out.dtype != x.dtype:
            raise ValueError("x and grad_out must share the plan dtype")
        shp = self.weight_grad_shape()
        if out is None:
            out = torch.empty(shp, dtype=torch.float32, device=x.device)
        if tuple(out.shape) != shp or out.dtype != torch.float32 or not out.is_contiguous():
            raise ValueError(f"grad_w must be a contiguous float32 tensor of shape {shp}")
        check(_lib.lib.fcfs_run_weight_grad(self._h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(grad_out.data_ptr()),
                                            ctypes.c_void_p(out.data_ptr()), N, self._stream(stream)),
              "fcfs_run_weight_grad")
        return out

    def run_rows(self, x_rows, in_row0: int, out_row0: int, out_nrows: int, out=None, stream=None):
        """Output rows [out_row0, out_row0+out_nrows) from input rows [in_row0, in_row0+x_rows.shape[2])."""
        import torch
        if len(self.dims) < 2:
            raise ValueError("row windows need a plan with rows (rank >= 2)")
        N, in_nrows = x_rows.shape[0], x_rows.shape[-2]
        self._check_tensor(x_rows, (N, self.C) + self.dims[:-2] + (in_nrows, self.W), "input rows")
        oshape = (N, self.C) + self.odims[:-2] + (out_nrows, self.Wo)
        if out is None:
            out = torch.empty(oshape, dtype=x_rows.dtype, device=x_rows.device)
        self._check_tensor(out, oshape, "output rows")
        check(_lib.lib.fcfs_run_rows(self._h, ctypes.c_void_p(x_rows.data_ptr()), in_row0, in_nrows,
                                     ctypes.c_void_p(out.data_ptr()), out_row0, out_nrows, N,
                                     self._stream(stream)), "fcfs_run_rows")
        return out

    def _check_host(self, t, shape, what):
        import torch
        if not isinstance(t, torch.Tensor) or t.device.type != "cpu":
            raise TypeError(f"{what} must be a CPU tensor")
        if _dtype_name(t.dtype) != self.dtype:
            raise TypeError(f"{what} dtype {t.dtype} does not match the plan's {self.dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{what} must be contiguous")
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{what} shape {tuple(t.shape)} != {tuple(shape)}")
        if not t.is_pinned():
            import warnings
            warnings.warn(f"{what} is not pinned: the copy is synchronous and slower", stacklevel=3)

    def run_host(self, x_host, out_host, dev_in, dev_out, stream=None):
        """End-to-end call with host buffers (fcfs_run_host): H2D copy of x_host
        into dev_in, the run into dev_out, D2H copy into out_host, all enqueued on
        the stream.  out_host holds the result only after that stream has
        synchronised.  Host tensors: contiguous CPU (pinned for async copies);
        device tensors: contiguous CUDA; all of the plan dtype and shapes."""
        N = x_host.shape[0]
        self._check_host(x_host, self.in_shape(N), "x_host")
        self._check_host(out_host, self.out_shape(N), "out_host")
        self._check_tensor(dev_in, self.in_shape(N), "dev_in")
        self._check_tensor(dev_out, self.out_shape(N), "dev_out")
        check(_lib.lib.fcfs_run_host(self._h, ctypes.c_void_p(x_host.data_ptr()), ctypes.c_void_p(out_host.data_ptr()),
                                     N, ctypes.c_void_p(dev_in.data_ptr()), ctypes.c_void_p(dev_out.data_ptr()),
                                     self._stream(stream)), "fcfs_run_host")
        return out_host


def last_launch() -> dict:
    """The calling thread's most recent launch (fcfs_last_launch): kernel and geometry."""
    import json
    buf = ctypes.create_string_buffer(1024)
    check(_lib.lib.fcfs_last_launch(buf, 1024), "fcfs_last_launch")
    return json.loads(buf.value.decode())


def kernel_launches() -> int:
    """Kernels the library has launched (or captured into graphs) in this process (fcfs_kernel_launches)."""
    return int(_lib.lib.fcfs_kernel_launches())


def run_batch(jobs, stream=None):
    """Run [(plan, x, out), ...] (independent jobs) with fcfs_run_batch: compatible
    jobs share kernel launches.  Outputs must be preallocated."""
    import torch
    arr = (_lib.Job * len(jobs))()
    for i, (pl, x, out) in enumerate(jobs):
        N = x.shape[0]
        pl._check_tensor(x, pl.in_shape(N), "input")
        pl._check_tensor(out, pl.out_shape(N), "output")
        arr[i] = _lib.Job(pl.handle.value, x.data_ptr(), out.data_ptr(), N)
    s = torch.cuda.current_stream() if stream is None else stream
    check(_lib.lib.fcfs_run_batch(ctypes.cast(arr, ctypes.c_void_p), len(jobs), ctypes.c_void_p(s.cuda_stream)),
          "fcfs_run_batch")
    return [out for _, _, out in jobs]


_cache: dict = {}
_cache_lock = threading.Lock()


def scale_nd(x, p, q, mode: str = "bilinear", pad: str = "replicate", extent: str = "paper", out=None,
             stream=None):
    """FCFS-resize the last len(p) axes of a CUDA tensor x (N, C, *dims) by the
    per-dimension factors p[d]/q[d] (§4.2): rank 1 (W), 2 (H, W) or 3 (D, H, W)."""
    import torch
    R = len(p)
    if x.dim() != R + 2:
        raise ValueError(f"expected an (N, C, {R} spatial dims) tensor, got shape {tuple(x.shape)}")
    x = x.contiguous()
    with torch.cuda.device(x.device):
        key = ("nd", tuple(p), tuple(q), mode, pad, x.shape[1], tuple(x.shape[2:]), _dtype_name(x.dtype), extent,
               x.device.index)
        with _cache_lock:
            pl = _cache.get(key)
            if pl is None:
                pl = Plan.nd(p, q, mode, pad, x.shape[1], tuple(x.shape[2:]), _dtype_name(x.dtype), extent)
                _cache[key] = pl
        return pl.run(x, out=out, stream=stream)


def _autograd_function():
    import torch

    class FCFSFunction(torch.autograd.Function):
        """y = FCFS(x) with its backward pass (fcfs_run_adjoint): the layer as a
        differentiable op inside a torch model (§7)."""

        @staticmethod
        def forward(ctx, x, plan):
            ctx.plan = plan
            return plan.run(x.contiguous())

        @staticmethod
        def backward(ctx, g):
            return ctx.plan.run_adjoint(g.contiguous()), None

    return FCFSFunction


_FCFS_FN = None


def apply(x, plan: Plan):
    """Differentiable FCFS: torch autograd calls the adjoint kernel in backward."""
    global _FCFS_FN
    if _FCFS_FN is None:
        _FCFS_FN = _autograd_function()
    return _FCFS_FN.apply(x, plan)


def get_plan(p, q, mode, pad, C, H, W, dtype, extent="paper", is1d=False, device=None) -> Plan:
    key = (p, q, mode, pad, C, H, W, dtype, extent, is1d, device)
    with _cache_lock:
        pl = _cache.get(key)
        if pl is None:
            pl = Plan(p, q, mode, pad, C, H, W, dtype, extent, is1d)
            _cache[key] = pl
    return pl


def scale(x, p: int, q: int, mode: str = "bilinear", pad: str = "replicate", extent: str = "paper",
          is1d: bool = False, out=None, stream=None):
    """FCFS-resize a CUDA tensor x of shape (N, C, H, W) (or (C, H, W), (H, W))
    by p/q.  Returns a new tensor (N, C, Ho, Wo) of x's dtype."""
    import torch
    squeeze = 0
    while x.dim() < 4:
        x = x.unsqueeze(0)
        squeeze += 1
    x = x.contiguous()
    with torch.cuda.device(x.device):
        pl = get_plan(p, q, mode, pad, x.shape[1], x.shape[2], x.shape[3], _dtype_name(x.dtype), extent, is1d,
                      x.device.index)
        y = pl.run(x, out=out, stream=stream)
    for _ in range(squeeze):
        y = y.squeeze(0)
    return y
