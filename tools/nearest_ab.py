"""A/B of nearest-gather variants (FCFS_DEBUG_NEAREST) on graph-timed steps: C2 (batched 2/3 + 3/4) and 2/1, 1/2 on 16x3x1024^2 (developer tool)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_10670_b200 as fc

def graph_us(fn, reps=50):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps): fn()
    with torch.cuda.stream(s):
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); g.replay(); e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps

res = {}
for v in sys.argv[1:]:
    os.environ["FCFS_DEBUG_NEAREST"] = v
    x = torch.rand(16, 3, 512, 512, device="cuda")
    a = fc.Plan(2, 3, "nearest", "zero", 3, 512, 512, "float32", "floor"); b = fc.Plan(3, 4, "nearest", "zero", 3, 512, 512, "float32", "floor")
    ya, yb = torch.empty(a.out_shape(16), device="cuda"), torch.empty(b.out_shape(16), device="cuda")
    t_c2 = graph_us(lambda: fc.run_batch([(a, x, ya), (b, x, yb)], stream=torch.cuda.current_stream()))
    x2 = torch.rand(16, 3, 1024, 1024, device="cuda")
    u = fc.Plan(2, 1, "nearest", "replicate", 3, 1024, 1024, "float32", "floor"); d = fc.Plan(1, 2, "nearest", "replicate", 3, 1024, 1024, "float32", "floor")
    yu, yd = torch.empty(u.out_shape(16), device="cuda"), torch.empty(d.out_shape(16), device="cuda")
    t_up = graph_us(lambda: u.run(x2, out=yu, stream=torch.cuda.current_stream()))
    t_dn = graph_us(lambda: d.run(x2, out=yd, stream=torch.cuda.current_stream()))
    print(f"variant {v}: C2 {t_c2:.2f} us, 2/1 {t_up:.2f} us, 1/2 {t_dn:.2f} us", flush=True)
