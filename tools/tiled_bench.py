"""Per-image time of the tiled kernel on the paper sweep's 27/11 and 2/11 factors (16 x 3 x 1024^2 fp32; developer tool)."""
import sys, torch
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_10670_b200 as fc
for (p, q, mode) in [(27, 11, "bilinear"), (27, 11, "bicubic"), (2, 11, "bilinear"), (2, 11, "bicubic")]:
    pl = fc.Plan(p, q, mode, "replicate", 3, 1024, 1024, "float32", "floor")
    xs = [torch.rand(16, 3, 1024, 1024, device="cuda") for _ in range(2)]
    outs = [torch.empty(pl.out_shape(16), device="cuda") for _ in range(2)]
    for i in range(3): pl.run(xs[i % 2], out=outs[i % 2])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(20): pl.run(xs[i % 2], out=outs[i % 2])
    e1.record(); torch.cuda.synchronize()
    print(p, q, mode, pl.kernel, round(e0.elapsed_time(e1) * 1e3 / 20 / 16, 2), "us/img")
