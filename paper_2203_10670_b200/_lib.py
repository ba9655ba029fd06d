"""ctypes binding of libfcfs.so (include/fcfs.h) -- argument marshalling only.

Every computation runs in the CUDA library.  If libfcfs.so is missing this
module raises at import: there is no CPU or PyTorch fallback.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FCFS_LIB", os.path.join(_PKG, "libfcfs.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libfcfs.so not found at {LIB_PATH}: build it with "
                      f"`python paper_2203_10670_b200/build.py` (there is no fallback path)")

lib = ctypes.CDLL(LIB_PATH)

i64, i32, u32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_uint, ctypes.c_void_p
P64 = ctypes.POINTER(ctypes.c_int64)


class Job(ctypes.Structure):
    _fields_ = [("plan", vp), ("in_", vp), ("out", vp), ("N", i64)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("p", i32), ("q", i32), ("mode", i32), ("pad", i32), ("dtype", i32), ("flags", u32),
                ("C", i64), ("H", i64), ("W", i64), ("Ho", i64), ("Wo", i64), ("ntaps", i32), ("lo", i32),
                ("kernel", i32), ("device", i32), ("in_rows_referenced", i64), ("rank", i32),
                ("pd", i32 * 3), ("qd", i32 * 3), ("dims", i64 * 3), ("odims", i64 * 3)]


# name -> (restype, argtypes); the ABI surface declared in include/fcfs.h
SIGNATURES = {
    "fcfs_plan_ex": (i32, [i32, i32, i32, i32, i64, i64, i64, i32, u32, ctypes.POINTER(vp)]),
    "fcfs_plan": (i32, [i32, i32, i32, i32, i64, i64, i64, i32, ctypes.POINTER(vp)]),
    "fcfs_plan_nd": (i32, [i32, ctypes.POINTER(i32), ctypes.POINTER(i32), i32, i32, i64, P64, i32, u32,
                           ctypes.POINTER(vp)]),
    "fcfs_output_dims": (i32, [vp, P64]),
    "fcfs_phase_table_dim": (i32, [vp, i32, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int)]),
    "fcfs_output_shape": (i32, [vp, P64, P64]),
    "fcfs_run": (i32, [vp, vp, vp, i64, vp]),
    "fcfs_run_rows": (i32, [vp, vp, i64, i64, vp, i64, i64, i64, vp]),
    "fcfs_run_rows_segments": (i32, [vp, i32, ctypes.POINTER(vp), P64, P64, vp, i64, i64, i64, vp]),
    "fcfs_run_batch": (i32, [vp, i32, vp]),
    "fcfs_strip_rows": (i32, [vp, i64, i64, P64, P64, P64, P64]),
    "fcfs_needed_rows": (i32, [vp, i64, i64, P64, P64]),
    "fcfs_run_host": (i32, [vp, vp, vp, i64, vp, vp, vp]),
    "fcfs_run_adjoint": (i32, [vp, vp, vp, i64, vp]),
    "fcfs_weight_grad_shape": (i32, [vp, P64]),
    "fcfs_run_weight_grad": (i32, [vp, vp, vp, vp, i64, vp]),
    "fcfs_plan_info": (i32, [vp, ctypes.POINTER(PlanInfo)]),
    "fcfs_launch_info": (i32, [vp, i64, i64, i64, ctypes.c_char_p, i64]),
    "fcfs_adjoint_info": (i32, [vp, i64, ctypes.c_char_p, i64]),
    "fcfs_last_launch": (i32, [ctypes.c_char_p, i64]),
    "fcfs_phase_table": (i32, [vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int)]),
    "fcfs_compulsory_bytes": (i32, [vp, i64, P64]),
    "fcfs_destroy": (None, [vp]),
    "fcfs_status_str": (ctypes.c_char_p, [i32]),
    "fcfs_version": (i32, []),
    "fcfs_kernel_launches": (ctypes.c_uint64, []),
}
for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

MODES = {"nearest": 0, "bilinear": 1, "bicubic": 2}
PADS = {"zero": 0, "replicate": 1, "reflect": 2}
DTYPES = {"float32": 0, "float16": 1, "bfloat16": 2}
FLAG_1D = 1 << 0
FLAG_EXTENT_FLOOR = 1 << 1
FLAG_FORCE_REFERENCE = 1 << 8
STATUS = {0: "FCFS_OK", 1: "FCFS_E_ARG", 2: "FCFS_E_SHAPE", 3: "FCFS_E_PAD", 4: "FCFS_E_UNSUPPORTED",
          5: "FCFS_E_DEVICE", 6: "FCFS_E_CUDA", 7: "FCFS_E_NOMEM"}
KERNELS = {0: "reference", 1: "nearest_gather", 2: "fused_separable", 3: "tiled"}


class FcfsError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = lib.fcfs_status_str(status).decode()
        super().__init__(f"{where}: {STATUS.get(status, status)} ({msg})")
        self.status = status
        self.name = STATUS.get(status, str(status))


def check(status: int, where: str) -> None:
    if status != 0:
        raise FcfsError(status, where)
