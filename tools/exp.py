"""Quick kernel-time experiments on the GPU (developer tool).

    python tools/exp.py C3 C4a C5 [--env FCFS_DEBUG_S=3,FCFS_DEBUG_S=4] [--reps 20]

For each launch config and each env setting: median CUDA-event time of one
fcfs_run over rotating buffers (> L2), achieved GB/s on algorithmic bytes.
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2203_10670_b200 as fc  # noqa: E402


def time_cfg(name, reps, env):
    for k in [k for k in os.environ if k.startswith("FCFS_DEBUG_") or k.startswith("FCFS_NO_")]:
        del os.environ[k]
    os.environ.update(env)
    import dataclasses
    hw = None
    if "@" in name:  # NAME@HxW: the config at another image size (2D configs)
        name, hw = name.split("@")
    c = synth.CONFIGS[name]
    if hw:
        h, w = (int(v) for v in hw.split("x"))
        c = dataclasses.replace(c, H=h, W=w)
    if c.nd:
        pl = fc.Plan.nd(c.pd, c.qd, c.mode, c.pad, c.C, c.dims, c.dtype, "floor")
    else:
        pl = fc.Plan(c.p, c.q, c.mode, c.pad, c.C, c.H, c.W, c.dtype, "floor", c.is1d)
    if c.wgrad:  # the weight gradient: (x, grad_out) -> grad_w
        x = synth.make_input(c).cuda()
        shp = pl.out_shape(c.N)
        g = torch.from_numpy(synth.normal_f32(c.seed + 7, int(np.prod(shp))).reshape(shp)).to(getattr(torch, c.dtype)).cuda()
        R = max(2, min(8, int(4 * 126e6 // ((x.numel() + g.numel()) * x.element_size())) + 1))
        xs = [x.clone() for _ in range(R)]
        gs = [g.clone() for _ in range(R)]
        gw = torch.empty(pl.weight_grad_shape(), device="cuda")
        fn = lambda i: pl.run_weight_grad(xs[i % R], gs[i % R], out=gw)
        for i in range(3):
            fn(i)
        torch.cuda.synchronize()
        ts = []
        for rep in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(reps):
                fn(i)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / reps)
        ts.sort()
        med = ts[len(ts) // 2]
        return med, (x.numel() + g.numel()) * x.element_size() / (med * 1e-6) / 1e9, {}
    if c.backward:  # the adjoint: grad_out -> grad_in
        shp = pl.out_shape(c.N)
        x = torch.from_numpy(synth.normal_f32(c.seed, int(np.prod(shp))).reshape(shp)).to(getattr(torch, c.dtype)).cuda()
        oshape, fn = pl.in_shape(c.N), pl.run_adjoint
    else:
        x = synth.make_input(c).cuda()
        oshape, fn = pl.out_shape(c.N), pl.run
    R = max(2, min(8, int(4 * 126e6 // (x.numel() * x.element_size() * 2)) + 1))
    xs = [x.clone() for _ in range(R)]
    ys = [torch.empty(oshape, dtype=x.dtype, device="cuda") for _ in range(R)]
    for i in range(3):
        fn(xs[i % R], out=ys[i % R])
    torch.cuda.synchronize()
    ts = []
    for rep in range(5):  # back-to-back launches (steady state), 5 batches
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(reps):
            fn(xs[i % R], out=ys[i % R])
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    ts.sort()
    med = ts[len(ts) // 2]
    by = (x.numel() + ys[0].numel()) * x.element_size() if c.backward else pl.compulsory_bytes(c.N)
    return med, by / (med * 1e-6) / 1e9, ({} if c.backward else pl.launch_info(c.N))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--env", default="")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    envs = [{}] + [dict(kv.split("=") for kv in e.split("+")) for e in a.env.split(",") if e]
    for name in a.configs:
        for env in envs:
            med, gbs, info = time_cfg(name, a.reps, env)
            keys = {k: info[k] for k in ("NS", "CPT", "ntile", "S", "flush_groups", "grid") if k in info}
            print(f"{name:4s} {str(env):34s} {med:9.1f} us {gbs:8.0f} GB/s {keys}", flush=True)
