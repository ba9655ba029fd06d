"""Seeded synthetic inputs for FCFS -- shared by tests (both sides) and bench.py.

This module holds none of the method's arithmetic: it only produces input
tensors with the shapes, dtypes and value distributions of BASELINE.json's
configs (recipe in DESIGN.md §4).  Generators are counter-based (splitmix64 of
(seed, global element index)) and implemented in ``synth.c``; any slice of a
batch or any row strip is bit-identical to slicing the full tensor.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "synth.c")
_LIB = os.path.join(_HERE, "libsynth.so")
_lock = threading.Lock()
_lib = None

SEED_BASE = 2203106700


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
                        "-o", tmp, _SRC, "-lm"], check=True)
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            u64, i64, fp = ctypes.c_uint64, ctypes.c_int64, ctypes.POINTER(ctypes.c_float)
            for name in ("synth_uniform_f32", "synth_uniform_f16grid", "synth_normal_f32"):
                getattr(lib, name).argtypes = [u64, i64, i64, fp]
            lib.synth_field_f32.argtypes = [u64, i64, i64, i64, i64, fp]
            lib.synth_hash.restype = u64
            lib.synth_hash.argtypes = [u64, u64]
            _lib = lib
    return _lib


def _fptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def hash64(seed: int, i: int) -> int:
    return _load().synth_hash(seed, i)


def uniform_f32(seed: int, n: int, off: int = 0) -> np.ndarray:
    out = np.empty(n, np.float32)
    _load().synth_uniform_f32(seed, off, n, _fptr(out))
    return out


def uniform_f16grid(seed: int, n: int, off: int = 0) -> np.ndarray:
    out = np.empty(n, np.float32)
    _load().synth_uniform_f16grid(seed, off, n, _fptr(out))
    return out


def normal_f32(seed: int, n: int, off: int = 0) -> np.ndarray:
    out = np.empty(n, np.float32)
    _load().synth_normal_f32(seed, off, n, _fptr(out))
    return out


def field_f32(seed: int, N: int, W: int, r0: int, r1: int) -> np.ndarray:
    out = np.empty((r1 - r0) * W, np.float32)
    _load().synth_field_f32(seed, N, W, r0, r1, _fptr(out))
    return out.reshape(r1 - r0, W)


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json workload (a single launch: one factor)."""
    name: str
    N: int
    C: int
    H: int
    W: int
    dtype: str          # "float32" | "float16" | "bfloat16"
    values: str         # "uniform" | "uniform_f16grid" | "normal" | "field"
    p: int
    q: int
    mode: str           # "nearest" | "bilinear" | "bicubic"
    pad: str            # "zero" | "replicate" | "reflect"
    floor_extent: bool = True
    is1d: bool = False
    seed: int = SEED_BASE
    D: int = 1                       # slices (3D volumes); the tensor is N x C x D x H x W
    pd: tuple | None = None          # per-dimension factors (outermost first): an ND plan (§4.2)
    qd: tuple | None = None
    backward: bool = False           # the adjoint launch: input = grad_out (N(0,1)), output = grad_in
    wgrad: bool = False              # the weight gradient: inputs x (the config's) and grad_out (N(0,1))

    @property
    def planes(self) -> int:
        return self.N * self.C

    @property
    def nd(self) -> bool:
        return self.pd is not None

    @property
    def dims(self) -> tuple:
        """spatial dims of the input tensor (after N, C)"""
        if not self.nd:
            return (self.H, self.W)
        return ((self.D,) if len(self.pd) == 3 else ()) + ((self.H,) if len(self.pd) >= 2 else ()) + (self.W,)


# BASELINE.json "configs" (index 0..4); a config with two factors is two launches.
CONFIGS = {
    "C1a": Config("C1a", 1, 1, 48, 64, "float32", "uniform", 3, 2, "bilinear", "replicate", seed=SEED_BASE + 1),
    "C1b": Config("C1b", 1, 1, 1, 101, "float32", "uniform", 2, 3, "nearest", "replicate", is1d=True,
                  seed=SEED_BASE + 11),
    "C2a": Config("C2a", 16, 3, 512, 512, "float32", "uniform", 2, 3, "nearest", "zero", seed=SEED_BASE + 2),
    "C2b": Config("C2b", 16, 3, 512, 512, "float32", "uniform", 3, 4, "nearest", "zero", seed=SEED_BASE + 2),
    "C3": Config("C3", 64, 64, 128, 128, "bfloat16", "normal", 5, 3, "bicubic", "reflect", seed=SEED_BASE + 3),
    "C4a": Config("C4a", 8, 3, 2160, 3840, "float16", "uniform_f16grid", 7, 5, "bilinear", "replicate",
                  seed=SEED_BASE + 4),
    "C4b": Config("C4b", 8, 3, 2160, 3840, "float16", "uniform_f16grid", 4, 7, "bilinear", "replicate",
                  seed=SEED_BASE + 4),
    "C5": Config("C5", 1, 1, 32768, 32768, "float32", "field", 3, 5, "bicubic", "replicate", seed=SEED_BASE + 5),
}

# Per-dimension factors and 3D volumes (not BASELINE.json
# configs): a 16:9 -> 4:3 width-only resize of config 4's frames (A1), a
# height-only bicubic 5/3 stretch of the same frames (A2), a trilinear
# 3/2 volume and a bicubic 5/3 bf16 feature volume.
CONFIGS.update({
    "A1": Config("A1", 8, 3, 2160, 3840, "float16", "uniform_f16grid", 3, 4, "bilinear", "replicate",
                 seed=SEED_BASE + 21, pd=(1, 3), qd=(1, 4)),
    "A2": Config("A2", 8, 3, 2160, 3840, "float16", "uniform_f16grid", 5, 3, "bicubic", "replicate",
                 seed=SEED_BASE + 24, pd=(5, 1), qd=(3, 1)),
    "V1": Config("V1", 4, 1, 256, 256, "float32", "uniform", 3, 2, "bilinear", "replicate", seed=SEED_BASE + 22,
                 D=128, pd=(3, 3, 3), qd=(2, 2, 2)),
    "V2": Config("V2", 2, 8, 128, 128, "bfloat16", "normal", 5, 3, "bicubic", "reflect", seed=SEED_BASE + 23,
                 D=64, pd=(5, 5, 5), qd=(3, 3, 3)),
})

# The backward pass of config 3: grad_in = A^T grad_out
# for the FCN feature-map resize, grad_out N(0,1) bf16 of the forward output shape.
CONFIGS["C3B"] = dataclasses.replace(CONFIGS["C3"], name="C3B", backward=True, seed=SEED_BASE + 31)
# ... and the gradient of its learnable taps (reading Z22): x of config 3 and a
# N(0,1) bf16 grad_out of the forward output shape -> 5 x 5 x 4 x 4 fp32
CONFIGS["C3W"] = dataclasses.replace(CONFIGS["C3"], name="C3W", wgrad=True, seed=SEED_BASE + 32)

# bench workloads: a step = one pass over one batch, every launch of the config
WORKLOADS = {
    "C1": ["C1a", "C1b"],
    "C2": ["C2a", "C2b"],
    "C3": ["C3"],
    "C4": ["C4a", "C4b"],
    "C5": ["C5"],
    "A1": ["A1"],
    "A2": ["A2"],
    "V1": ["V1"],
    "V2": ["V2"],
    "C3B": ["C3B"],
    "C3W": ["C3W"],
}


def make_values(cfg: Config, n0: int = 0, n1: int | None = None, rows: tuple[int, int] | None = None,
                batch_offset: int = 0) -> np.ndarray:
    """float32 numpy array (n1-n0, C, r1-r0, W) of the config's values (before
    the cast to cfg.dtype).  batch_offset shifts the global batch index (a rank's
    own batch in weak scaling)."""
    n1 = cfg.N if n1 is None else n1
    r0, r1 = (0, cfg.H) if rows is None else rows
    nb = n1 - n0
    if cfg.values == "field":
        assert cfg.N == 1 and cfg.C == 1
        return field_f32(cfg.seed + batch_offset, cfg.H, cfg.W, r0, r1).reshape(1, 1, r1 - r0, cfg.W)
    gen = {"uniform": uniform_f32, "uniform_f16grid": uniform_f16grid, "normal": normal_f32}[cfg.values]
    plane = cfg.D * cfg.H * cfg.W
    if (r0, r1) == (0, cfg.H):  # contiguous global index range
        off = (batch_offset + n0) * cfg.C * plane
        return gen(cfg.seed, nb * cfg.C * plane, off).reshape((nb, cfg.C) + cfg.dims)
    assert cfg.D == 1
    out = np.empty((nb, cfg.C, r1 - r0, cfg.W), np.float32)
    for b in range(nb):
        for c in range(cfg.C):
            gplane = (batch_offset + n0 + b) * cfg.C + c
            out[b, c] = gen(cfg.seed, (r1 - r0) * cfg.W, gplane * plane + r0 * cfg.W).reshape(r1 - r0, cfg.W)
    return out


def make_input(cfg: Config, n0: int = 0, n1: int | None = None, rows=None, batch_offset: int = 0):
    """torch CPU tensor of dtype cfg.dtype (fp32 values rounded RNE)."""
    import torch
    v = torch.from_numpy(make_values(cfg, n0, n1, rows, batch_offset))
    return v.to(getattr(torch, cfg.dtype))
