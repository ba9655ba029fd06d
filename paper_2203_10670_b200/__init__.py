"""B200-native FCFS (arXiv 2203.10670): fractional p/q scaling as one fused
pad -> strided polyphase conv -> pixelshuffle pass (libfcfs.so, sm_100a).

Public API:
    scale(x, p, q, mode, pad, extent, is1d)  -- resize a CUDA tensor (one factor, 2D or rows)
    scale_nd(x, (p..), (q..), mode, pad)     -- per-dimension factors, rank 1-3 (§4.2)
    Plan(...)                                 -- an explicit plan (run / run_rows / run_host / run_adjoint /
                                                 run_weight_grad)
    apply(x, plan)                            -- differentiable (torch autograd; backward = the adjoint kernel)
    dist                                      -- multi-GPU drivers (batch shards, row strips + NCCL halo)
"""
from ._lib import FcfsError, LIB_PATH  # noqa: F401  (raises ImportError if libfcfs.so is missing)
from .fcfs import Plan, apply, get_plan, kernel_launches, last_launch, run_batch, scale, scale_nd  # noqa: F401

__all__ = ["Plan", "apply", "get_plan", "kernel_launches", "last_launch", "run_batch", "scale", "scale_nd", "FcfsError", "LIB_PATH"]
