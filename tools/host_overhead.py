"""Host-side cost of eager Plan.run calls on tiny images (ctypes marshalling + planning; developer tool)."""
import time, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_10670_b200 as fc
for (p, q, mode, dtype, H, W) in [(5, 3, "bicubic", "bfloat16", 64, 64), (2, 3, "nearest", "float32", 64, 64), (27, 11, "bilinear", "float32", 64, 64)]:
    pl = fc.Plan(p, q, mode, "replicate", 1, H, W, dtype, "floor")
    x = torch.rand(1, 1, H, W, device="cuda").to(getattr(torch, dtype)); y = pl.run(x)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    t0 = time.perf_counter()
    for _ in range(2000): pl.run(x, out=y, stream=s)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(pl.kernel, f"host {1e6*(t1-t0)/2000:.1f} us/call, total {1e6*(t2-t0)/2000:.1f} us/call")
