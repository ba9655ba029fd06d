"""Diagnose fused-vs-reference mismatches on the GPU (developer tool)."""
import itertools
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2203_10670_b200 as fc  # noqa: E402

DEV = "cuda:0"


def rand(seed, shape, dtype):
    v = synth.normal_f32(seed, int(np.prod(shape))).reshape(shape)
    return torch.from_numpy(v).to(getattr(torch, dtype)).to(DEV)


def diff(case, env):
    (p, q, mode, pad, dtype, N, C, H, W, ext) = case
    for k in ("FCFS_DEBUG_NBANDS", "FCFS_DEBUG_GRID", "FCFS_DEBUG_S"):
        os.environ.pop(k, None)
    os.environ.update(env)
    x = rand(11, (N, C, H, W), dtype)
    pl = fc.Plan(p, q, mode, pad, C, H, W, dtype, ext)
    y = pl.run(x)
    yr = fc.Plan(p, q, mode, pad, C, H, W, dtype, ext, force_reference=True).run(x)
    torch.cuda.synchronize()
    bad = (y.view(torch.int16 if dtype != "float32" else torch.int32) !=
           yr.view(torch.int16 if dtype != "float32" else torch.int32))
    nb = int(bad.sum())
    msg = f"{case} env={env} kernel={pl.kernel} mismatches={nb}/{bad.numel()}"
    if nb:
        idx = bad.nonzero().cpu().numpy()
        planes = sorted(set((idx[:, 0] * C + idx[:, 1]).tolist()))
        rows = sorted(set(idx[:, 2].tolist()))
        cols = sorted(set(idx[:, 3].tolist()))
        msg += f"\n   planes={planes[:20]} rows={rows[:40]} cols({len(cols)})={cols[:40]}"
    print(msg, flush=True)
    return nb


if __name__ == "__main__":
    os.environ["FCFS_DEBUG_PRINT"] = "1"
    cases = [
        (3, 2, "bilinear", "zero", "bfloat16", 1, 3, 8, 104, "floor"),
        (3, 2, "bilinear", "zero", "float32", 1, 3, 8, 104, "floor"),
        (3, 2, "bilinear", "replicate", "bfloat16", 1, 3, 8, 104, "floor"),
        (5, 3, "bicubic", "reflect", "bfloat16", 2, 3, 64, 128, "floor"),
        (5, 3, "bicubic", "reflect", "float32", 2, 3, 64, 128, "floor"),
        (5, 3, "bicubic", "reflect", "bfloat16", 1, 1, 64, 128, "floor"),
    ]
    for case in cases:
        for env in ({}, {"FCFS_DEBUG_NBANDS": "1"}, {"FCFS_DEBUG_GRID": "1"}, {"FCFS_DEBUG_S": "2"},
                    {"FCFS_DEBUG_NBANDS": "1", "FCFS_DEBUG_GRID": "1"}):
            diff(case, env)
