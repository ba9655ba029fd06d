#!/usr/bin/env python
"""FCFS hot-path benchmark (BASELINE.json metric: output Mpix/s and achieved
HBM GB/s vs 8 TB/s, 1/2/4/8 B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C2] [--impl fcfs|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one process per GPU, NCCL)

A step is one pass of the whole hot path over one batch: every launch of the
workload.  The default workload is C5 (BASELINE.json configs[4]: one
32768^2 fp32 image, bicubic 3/5), the largest single-GPU configuration: the
metric names no config, so the headline is measured on the largest one.  At
N > 1 C5 shards by row strips with an NCCL halo exchange (strong scaling,
paper_2203_10670_b200.dist); batched workloads (C2 16, C3 64, C4 8 images)
give each rank its share of the batch (--split batch, strong scaling, no
data-path collective) or a whole batch of its own (--split weak).

Prints ONE JSON line on rank 0.  Inputs are resident in HBM before the timed
region; between steps the input/output buffers rotate over a set larger than
4x L2, so no step reads its input from L2.  Times are CUDA events on the
launching stream, max over ranks.
"""
from __future__ import annotations

import argparse
import dataclasses
import datetime
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "FCFS resize output Mpix/s per GPU and achieved HBM GB/s vs 8 TB/s, 1/2/4/8 B200"
DTYPE_TAG = {"float32": "f32", "float16": "f16", "bfloat16": "bf16"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="C5", choices=sorted(synth.WORKLOADS))
    ap.add_argument("--split", default="batch", choices=["batch", "weak"],
                    help="batched workloads at N > 1: 'batch' gives rank r its share of the config's N images "
                         "(SURVEY 8(e), strong scaling); 'weak' gives every rank a whole batch of its own")
    ap.add_argument("--impl", default="fcfs", choices=["fcfs", "reference"])
    ap.add_argument("--soak-s", type=float, default=1.0, help="untimed steady-state run before warm-up (clocks)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cold", action="store_true", help="skip the cold-L2 single-step median/min (SURVEY 8d)")
    ap.add_argument("--cold-reps", type=int, default=100)
    ap.add_argument("--halo", default="nccl", choices=["nccl", "peer"],
                    help="C5 row strips at N > 1: NCCL send/recv halo, or in-kernel peer reads (symmetric memory)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-strips", action="store_true", help="C5: the row-strip path even at N = 1 (testing)")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the run."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.marks = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.idx)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, name):
        self.marks.append((name, time.time()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0, t1):
        rows = []
        for ts, line in self.lines:
            if t0 - 0.15 <= ts <= t1 + 0.15:
                f = [x.strip() for x in line.split(",")]
                if len(f) >= 9:
                    rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())}


def batch_share(n: int, rank: int, world: int):
    """Images [a, b) of an n-image batch that rank `rank` of `world` scales
    (--split batch): contiguous, disjoint, covering [0, n)."""
    return rank * n // world, (rank + 1) * n // world


def provenance():
    """What ran where: the git commit when the tree has one (gpurun copies omit
    .git), a hash of the product sources and bench.py, the host CPU."""
    import glob
    import hashlib
    out = {}
    try:
        out["git_sha"] = subprocess.run(["git", "-C", ROOT, "rev-parse", "HEAD"], capture_output=True, text=True,
                                        timeout=10).stdout.strip() or None
    except Exception:
        out["git_sha"] = None
    h = hashlib.sha256()
    files = sorted(glob.glob(os.path.join(ROOT, "paper_2203_10670_b200", "csrc", "*")) +
                   glob.glob(os.path.join(ROOT, "include", "*.h")) + [os.path.join(ROOT, "bench.py")])
    for f in files:
        with open(f, "rb") as fh:
            h.update(os.path.basename(f).encode() + fh.read())
    out["src_sha16"] = h.hexdigest()[:16]
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    out["host_cpu"] = {"model": model, "cores": os.cpu_count()}
    return out


def physical_gpu_index(local_rank: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        try:
            return int(vis.split(",")[local_rank])
        except Exception:
            return local_rank
    return local_rank


# --------------------------------------------------------------------------- CPU oracle leg
def oracle_sample_run(cfgs, planes_per_cfg: int, keep: list | None = None):
    """Run the oracle (staged, as it stands) on `planes_per_cfg` planes of every
    launch of the workload; returns (outputs, seconds, description).  keep: a
    list that receives (config name, what, oracle result) of every sample, for
    the parity check of the GPU result on the same sample."""
    import numpy as np
    import oracle
    outs, secs, parts = 0, 0.0, []
    for cfg in cfgs:
        n_img = max(1, min(cfg.N, -(-planes_per_cfg // cfg.C)))
        if cfg.backward or cfg.wgrad:  # the oracle's adjoint / weight gradient on whole planes
            n_img = max(1, min(cfg.N, -(-planes_per_cfg // cfg.C)))
            pl_sh = (n_img, cfg.C) + tuple(oracle.output_dims_nd(cfg.dims, (cfg.p,) * 2, (cfg.q,) * 2,
                                                                 cfg.floor_extent))
            g = synth.normal_f32(cfg.seed, int(np.prod(pl_sh))).reshape(pl_sh)
            t0 = time.perf_counter()
            if cfg.backward:
                y = oracle.adjoint_nd(g, cfg.dims, (cfg.p,) * 2, (cfg.q,) * 2, cfg.mode, cfg.pad, cfg.floor_extent)
            else:
                x = synth.make_values(cfg, 0, n_img)
                y = oracle.weight_grad(x, g, cfg.p, cfg.q, cfg.mode, cfg.pad, floor_extent=cfg.floor_extent)
            secs += time.perf_counter() - t0
            if keep is not None and cfg.backward:
                keep.append((cfg.name, ("images", 0, n_img), y))
            outs += g.size
            parts.append(f"{cfg.name}: {'adjoint' if cfg.backward else 'weight gradient'} of "
                         f"{n_img * cfg.C} of {cfg.planes} planes")
            continue
        if cfg.values == "field":
            rows = (0, min(cfg.H, 600))
            x = synth.make_values(cfg, 0, 1, rows=rows)
            # output rows whose whole hidden-row window lies inside the sampled input rows
            Ho_rows = (0, ((rows[1] - 2 * cfg.q - 4) // cfg.q) * cfg.p)
            t0 = time.perf_counter()
            y = oracle.staged(x[0], cfg.p, cfg.q, cfg.mode, cfg.pad, floor_extent=True, rows=Ho_rows, H=cfg.H)
            secs += time.perf_counter() - t0
            if keep is not None:
                keep.append((cfg.name, ("rows",) + Ho_rows, y))
            outs += y.size
            parts.append(f"{cfg.name}: output rows {Ho_rows[0]}..{Ho_rows[1]} of 1 plane")
            continue
        x = synth.make_values(cfg, 0, n_img)
        t0 = time.perf_counter()
        if cfg.nd:
            y = oracle.staged_nd(x, cfg.pd, cfg.qd, cfg.mode, cfg.pad, floor_extent=cfg.floor_extent)
        else:
            y = oracle.staged(x, cfg.p, cfg.q, cfg.mode, cfg.pad, floor_extent=cfg.floor_extent, is1d=cfg.is1d)
        secs += time.perf_counter() - t0
        if keep is not None:
            keep.append((cfg.name, ("images", 0, n_img), y))
        outs += y.size
        parts.append(f"{cfg.name}: {n_img * cfg.C} of {cfg.planes} planes")
    return outs, secs, "; ".join(parts)


def cpu_baseline(cfgs, budget_s=10.0, gpu_result=None):
    """The oracle as it stands on this host's cores: a sample of the workload
    grown (then repeated) until it has run about budget_s seconds.

    gpu_result(config name, what) -> the timed GPU path's output on the same
    sample (a CPU tensor): the line then also carries the sample's parity
    against the oracle (BASELINE.json bar; the tests check every output)."""
    cores = os.cpu_count() or 1
    planes = max(1, cores)
    keep = []
    outs, secs, desc = oracle_sample_run(cfgs, planes, keep)
    while secs < budget_s / 8 and not all(planes >= c.planes for c in cfgs):
        planes *= 4
        keep = []
        outs, secs, desc = oracle_sample_run(cfgs, planes, keep)
    tot_o, tot_s, reps = outs, secs, 1
    while tot_s < budget_s and reps < 1000:
        o, s, _ = oracle_sample_run(cfgs, planes)
        tot_o += o
        tot_s += s
        reps += 1
    threads = 1 if all(c.wgrad for c in cfgs) else cores  # the weight-gradient oracle is single-threaded
    res = {"value": tot_o / tot_s / 1e6, "unit": "Mpix/s", "cores": threads, "kind": "oracle",
           "sample": f"C oracle (double, {threads} thread{'s' if threads > 1 else ''}) on {desc}, {reps} passes; "
                     f"{tot_s:.1f} s"}
    if gpu_result is not None and keep:
        res["parity"] = [sample_parity(cfg_by_name(cfgs, name), what, ref, gpu_result(name, what))
                         for name, what, ref in keep]
    return res


def cfg_by_name(cfgs, name):
    return next(c for c in cfgs if c.name == name)


def sample_parity(cfg, what, ref, gpu):
    """The GPU output of one oracle sample against the BASELINE.json bar:
    nearest bit-exact, fp32 max abs error <= 1e-5 x input range, 16-bit
    ordered-ulp distance from the oracle rounded to the dtype (elements > 1 ulp
    counted; the tests apply reading Z18 to those)."""
    import numpy as np
    import torch
    import oracle
    gpu, x_range = gpu
    ref = np.asarray(ref, dtype=np.float64)
    if what[0] == "images" and gpu.shape[0] < ref.shape[0]:  # a rank's share of the batch holds fewer images
        ref = ref[:gpu.shape[0]]
    ref = ref.reshape(tuple(gpu.shape))
    out = {"config": cfg.name, "sample": list(what), "outputs": int(ref.size)}
    if cfg.backward:
        out.update(max_abs_err=float(np.abs(gpu.double().numpy() - ref).max()), max_abs_ref=float(np.abs(ref).max()))
        return out
    if cfg.dtype == "float32":
        r = torch.from_numpy(ref.astype(np.float32))
    else:
        r = oracle.round_to(ref, cfg.dtype)
        r = r if isinstance(r, torch.Tensor) else torch.from_numpy(r)
    ib = torch.int32 if cfg.dtype == "float32" else torch.int16
    if cfg.mode == "nearest":
        n = int((gpu.contiguous().view(ib) != r.contiguous().view(ib)).sum())
        out.update(bit_mismatches=n, within_bar=n == 0)
        return out
    err = float(np.abs(gpu.double().numpy() - ref).max())
    out["max_abs_err"] = err
    if cfg.dtype == "float32":
        tol = 1e-5 * x_range
        out.update(tol=tol, within_bar=err <= tol)
        return out

    def ordered(t):
        b = t.contiguous().view(torch.int16).numpy().astype(np.int32) & 0xFFFF
        return np.where(b & 0x8000, -(b & 0x7FFF), b & 0x7FFF)
    d = np.abs(ordered(gpu) - ordered(r))
    out.update(max_ulp=int(d.max()), over_1ulp=int((d > 1).sum()))
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfgs = [synth.CONFIGS[n] for n in synth.WORKLOADS[args.workload]]
    cores = os.cpu_count() or 1
    planes = max(1, cores)
    for _ in range(args.warmup):
        oracle_sample_run(cfgs, planes)
    tot_o, tot_s, desc = 0, 0.0, ""
    for _ in range(args.steps):
        o, s, desc = oracle_sample_run(cfgs, planes)
        tot_o += o
        tot_s += s
    value = tot_o / tot_s / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "Mpix/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_s / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": DTYPE_TAG[cfgs[0].dtype], "data": "synthetic",
            "config": {"workload": args.workload, "launches": [c.name for c in cfgs]},
            "cpu_baseline": {"value": value, "unit": "Mpix/s",
                             "cores": 1 if all(c.wgrad for c in cfgs) else cores, "kind": "oracle",
                             "sample": f"each step: {desc}"},
            "e2e": {"value": value, "unit": "Mpix/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if args.workload == "C1":  # the 1-thread oracle time of config 0 ("well under a second")
        import oracle
        one = {}
        for c in cfgs:
            x = synth.make_values(c)
            t0 = time.perf_counter()
            oracle.staged(x, c.p, c.q, c.mode, c.pad, floor_extent=c.floor_extent, is1d=c.is1d, nthreads=1)
            one[c.name] = time.perf_counter() - t0
        line["oracle_1thread_s"] = one
    print(json.dumps(line), flush=True)
    return 0


def kernel_name(L):
    if L["cfg"].backward:
        return "fused_adjoint (+ border bands for replicate/reflect)"
    if L["cfg"].wgrad:
        return "weight_grad"
    return L["plan"].launch_info(L["cfg"].N)["kernel"]  # the variant fcfs_run launches (fused_plane, ...)


def make_plan(fc, cfg):
    ext = "floor" if cfg.floor_extent else "paper"
    if cfg.nd:
        return fc.Plan.nd(cfg.pd, cfg.qd, cfg.mode, cfg.pad, cfg.C, cfg.dims, cfg.dtype, ext)
    return fc.Plan(cfg.p, cfg.q, cfg.mode, cfg.pad, cfg.C, cfg.H, cfg.W, cfg.dtype, ext, cfg.is1d)


# --------------------------------------------------------------------------- GPU leg
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(minutes=10))
    import paper_2203_10670_b200 as fc

    cfgs = [synth.CONFIGS[n] for n in synth.WORKLOADS[args.workload]]
    if args.workload == "C5" and (world > 1 or args.force_strips):
        return bench_strips(args, cfgs[0], rank, world, dev)
    # --split batch (N > 1): rank r scales images [r N / G, (r + 1) N / G) of the
    # config's batch; --split weak: a whole batch of its own
    split = world > 1 and args.split == "batch"

    stream = torch.cuda.Stream(dev)  # every launch of the run goes to this stream (also the graph capture stream)
    props = torch.cuda.get_device_properties(dev)
    l2 = getattr(props, "L2_cache_size", 126 * 2 ** 20) or 126 * 2 ** 20
    launches = []
    for gcfg in cfgs:
        cfg = gcfg
        img0, img1 = 0, gcfg.N
        if split:
            img0, img1 = batch_share(gcfg.N, rank, world)
            if img1 <= img0:
                raise SystemExit(f"--split batch: {gcfg.name} has {gcfg.N} images for {world} ranks")
            cfg = dataclasses.replace(gcfg, N=img1 - img0)
        pl = make_plan(fc, cfg)
        if cfg.backward:  # the adjoint: grad_out (forward output shape) -> grad_in (forward input shape)
            shp = pl.out_shape(cfg.N)
            n = 1
            for d in shp:
                n *= d
            x = torch.from_numpy(synth.normal_f32(cfg.seed + rank, n).reshape(shp)).to(getattr(torch, cfg.dtype))
            oshape = pl.in_shape(cfg.N)
        else:
            x = (synth.make_input(gcfg, img0, img1) if split else
                 synth.make_input(cfg, batch_offset=rank * cfg.N))
            oshape = pl.out_shape(cfg.N)
        n_out = 1
        for d in oshape:
            n_out *= d
        nbytes = (x.numel() + n_out) * x.element_size() if cfg.backward else pl.compulsory_bytes(cfg.N)
        g_host = None
        if cfg.wgrad:  # weight gradient: inputs x and grad_out (the output's shape); "outputs" = grad_out pixels
            g_host = torch.from_numpy(synth.normal_f32(cfg.seed + 7 + rank, n_out).reshape(oshape)).to(
                getattr(torch, cfg.dtype))
            nbytes = (x.numel() + n_out) * x.element_size()
        launches.append({"cfg": cfg, "plan": pl, "x_host": x, "bytes": nbytes, "outputs": n_out, "oshape": oshape,
                         "g_host": g_host})
    # input/output buffers per rotation set; several launches may share one input
    set_bytes = 0
    host_inputs = {}
    for L in launches:
        key = (L["cfg"].seed, L["cfg"].N, L["cfg"].H, L["cfg"].W, L["cfg"].dtype)
        if key not in host_inputs:
            host_inputs[key] = L["x_host"]
            set_bytes += L["x_host"].numel() * L["x_host"].element_size()
        L["key"] = key
        set_bytes += L["outputs"] * L["x_host"].element_size()
    R = max(2, min(64, -(-4 * l2 // set_bytes)))
    free = torch.cuda.mem_get_info(dev)[0]
    R = max(1, min(R, int(0.8 * free // set_bytes)))
    dev_inputs = {k: [v.to(dev) for _ in range(R)] for k, v in host_inputs.items()}
    for L in launches:
        if L["cfg"].wgrad:
            L["g_dev"] = [L["g_host"].to(dev) for _ in range(R)]
            L["outs"] = [torch.empty(L["plan"].weight_grad_shape(), dtype=torch.float32, device=dev) for _ in range(R)]
        else:
            L["outs"] = [torch.empty(L["oshape"], dtype=L["x_host"].dtype, device=dev) for _ in range(R)]
    torch.cuda.synchronize(dev)

    # kernel launches of a step: nearest-gather launches of one dtype share one
    # launch (fcfs_run_batch); every other launch is its own group
    if len(launches) > 1 and all(L["plan"].kernel == "nearest_gather" for L in launches):
        groups = [list(range(len(launches)))]
    else:
        groups = [[i] for i in range(len(launches))]

    def step(r, only=None):
        for gi, grp in enumerate(groups):
            if only is not None and gi != only:
                continue
            if len(grp) == 1:
                L = launches[grp[0]]
                if L["cfg"].backward:
                    L["plan"].run_adjoint(dev_inputs[L["key"]][r], out=L["outs"][r], stream=stream)
                elif L["cfg"].wgrad:
                    L["plan"].run_weight_grad(dev_inputs[L["key"]][r], L["g_dev"][r], out=L["outs"][r], stream=stream)
                else:
                    L["plan"].run(dev_inputs[L["key"]][r], out=L["outs"][r], stream=stream)
            else:
                fc.run_batch([(launches[i]["plan"], dev_inputs[launches[i]["key"]][r], launches[i]["outs"][r])
                              for i in grp], stream=stream)

    def capture(nsteps, only=None):
        """CUDA graph of nsteps steps over the rotating buffer sets (launch-bound
        host path removed: the graph replays the library's kernel launches)."""
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for s_ in range(nsteps):
                step(s_ % R, only)
        return g

    def timed_replay(g):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.replay()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1)

    sampler = ClockSampler(physical_gpu_index(local))
    sampler.start()
    t_soak0 = time.time()
    k = 0
    while time.time() - t_soak0 < args.soak_s:
        for _ in range(50):
            step(k % R)
            k += 1
        torch.cuda.synchronize(dev)
    for w in range(args.warmup):  # eager warm-up (also configures the kernels)
        step(w % R)
    torch.cuda.synchronize(dev)
    n_launch0 = fc.kernel_launches()
    graph = capture(args.steps)
    n_launches = fc.kernel_launches() - n_launch0  # the library's kernels captured in the timed graph
    with torch.cuda.stream(stream):
        graph.replay()  # graph warm-up (upload)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t_wall0 = time.time()
    with torch.cuda.stream(stream):
        elapsed_ms = timed_replay(graph)
    t_wall1 = time.time()
    if world > 1:
        dist.barrier()
    # average launch duration of each kernel group: the timed region itself when
    # a step is one launch, else a graph of K back-to-back launches of that group
    if len(groups) == 1:
        per_group_ms = [elapsed_ms / args.steps]
    else:
        per_group_ms = []
        for gi in range(len(groups)):
            gg = capture(args.steps, only=gi)
            with torch.cuda.stream(stream):
                gg.replay()
                torch.cuda.synchronize(dev)
                per_group_ms.append(timed_replay(gg) / args.steps)
            del gg
    if world > 1:
        t = torch.tensor([elapsed_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    clocks = sampler.summary(t_soak0, t_wall1)
    sampler.stop()

    outputs_per_step = sum(L["outputs"] for L in launches)
    total_outputs = outputs_per_step * world  # every rank's outputs of one step (uneven batch shares summed)
    if world > 1:
        t = torch.tensor([outputs_per_step], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        total_outputs = float(t.item())
    # algorithmic bytes of a launch group: every output byte once plus every
    # input row some job of the group reads once (jobs of one launch that scale
    # the same input share its rows: C2a and C2b read the batch once)
    def group_bytes(grp):
        tot = sum(launches[i]["outputs"] * launches[i]["x_host"].element_size() for i in grp)
        by_key = {}
        for i in grp:
            by_key.setdefault(launches[i]["key"], []).append(i)
        for key, idx in by_key.items():
            L0 = launches[idx[0]]
            row_b = L0["cfg"].N * L0["cfg"].C * L0["cfg"].W * L0["x_host"].element_size()
            if len(idx) == 1:
                tot += L0["bytes"] - L0["outputs"] * L0["x_host"].element_size()
            else:
                rows = set()
                for i in idx:
                    pl = launches[i]["plan"]
                    assert pl.kernel == "nearest_gather"
                    rows |= {(m * pl.q) // pl.p for m in range(pl.Ho)}
                tot += len(rows) * row_b
        return tot

    bytes_per_step = sum(group_bytes(g) for g in groups)
    ms_per_step = elapsed_ms / args.steps
    value = total_outputs * args.steps / (elapsed_ms * 1e-3) / 1e6
    peak, peak_kind = peaks()
    dom = max(range(len(groups)), key=lambda gi: per_group_ms[gi])  # dominant kernel launch
    dom_ms = per_group_ms[dom]
    dom_name = "+".join(launches[i]["cfg"].name for i in groups[dom])
    dom_bytes = group_bytes(groups[dom])
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic = tj.get(dom_name)
    except Exception:
        pass

    # SURVEY §8(d) single-launch protocol: cold L2 (a > L2 buffer written before
    # each repeat), CUDA events around one eager step, median and min
    cold = None
    if not args.no_cold:
        flush = torch.empty(int(2 * l2) // 4, dtype=torch.float32, device=dev)
        ts = []
        with torch.cuda.stream(stream):
            for r in range(args.cold_reps):
                flush.fill_(float(r))
                c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                c0.record(stream)
                step(r % R)
                c1.record(stream)
                c1.synchronize()
                ts.append(c0.elapsed_time(c1) * 1e3)
        del flush
        ts.sort()
        cold = {"median_us": ts[len(ts) // 2], "min_us": ts[0], "repeats": len(ts),
                "protocol": "L2 flushed (2x L2 written) before each repeat; CUDA events around one eager step"}

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(launches, args, dev, stream, world, dist, fc=fc, groups=groups, total_outputs=total_outputs)

    line = {
        "metric": METRIC, "value": value, "unit": "Mpix/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if split else "weak",
        "vs_baseline": None, "dtype": DTYPE_TAG[cfgs[0].dtype], "data": "synthetic",
        "config": {"workload": args.workload, "launches": [
            {"name": L["cfg"].name, "shape": [L["cfg"].N, L["cfg"].C, *L["cfg"].dims],
             "factor": (f"{L['cfg'].p}/{L['cfg'].q}" if not L["cfg"].nd else
                        " x ".join(f"{a}/{b}" for a, b in zip(L["cfg"].pd, L["cfg"].qd))),
             "mode": L["cfg"].mode, "pad": L["cfg"].pad,
             "dtype": L["cfg"].dtype, "out": list(L["plan"].odims), "kernel": kernel_name(L),
             "compulsory_bytes_alone": L["bytes"],
             "avg_launch_us": per_group_ms[next(gi for gi, g in enumerate(groups) if i in g)] * 1e3,
             "shares_launch_with": [launches[j]["cfg"].name for g in groups if i in g for j in g if j != i]}
            for i, L in enumerate(launches)],
            "launch_info": [dict(launches[g[0]]["plan"].launch_info(launches[g[0]]["cfg"].N),
                                 jobs=[launches[i]["cfg"].name for i in g]) for g in groups],
            "per_rank_batch": (f"rank {rank}: images of the config's batch split {world} ways (strong scaling)"
                               if split else "own batch per rank (weak scaling)"),
            "l2": f"rotating {R} buffer sets of {set_bytes / 2**20:.0f} MiB (> 4x {l2 / 2**20:.0f} MiB L2); no flush",
            "soak_s": args.soak_s, "parallelism": f"dp{world}",
            "timing": "CUDA graph of K steps replayed once between CUDA events (steady-state launches)"},
        "per_gpu_mpix_s": value / world,
        "achieved_GBps_step": bytes_per_step / (ms_per_step * 1e-3) / 1e9,
        "frac_of_8TBps_step": bytes_per_step / (ms_per_step * 1e-3) / 8e12,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": kernel_name(launches[groups[dom][0]]), "launch": dom_name,
                     "peak_source": f"{peak_kind} MEASURED_PEAKS.json hbm_gbs" if peak_kind == "measured" else
                     "fallback 6.65 TB/s (B200_PROFILING.md)",
                     "algorithmic_bytes_per_launch": dom_bytes, "avg_launch_us": dom_ms * 1e3,
                     "timing": ("timed region: CUDA events around one CUDA-graph replay of exactly K steps "
                                "(the library's launches captured on the launching stream); per-launch average = "
                                "region / K when a step is one launch, else a graph of K launches of that kernel")},
        "gpu_launches": n_launches,
        "single_launch_cold_l2": cold,
        "clocks": clocks,
        "provenance": provenance(),
    }
    if e2e is not None:
        line["e2e"] = e2e
    if rank == 0 and not args.no_cpu_baseline:
        def gpu_result(name, what):
            L = next(L for L in launches if L["cfg"].name == name)
            o = L["outs"][0]  # every rotation set holds the same input, so any set's output
            x = dev_inputs[L["key"]][0]
            rng = float((x.max() - x.min()).float().item()) if not L["cfg"].wgrad else 1.0
            if what[0] == "rows":
                return o[:, :, what[1]:what[2]].cpu(), rng
            return o[what[1]:min(what[2], o.shape[0])].cpu(), rng
        line["cpu_baseline"] = cpu_baseline(cfgs, gpu_result=gpu_result)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def bench_strips(args, cfg, rank, world, dev):
    """--workload C5 at N > 1 (or --force-strips): the 32768^2 image in row
    strips (paper_2203_10670_b200.dist.StripRunner), the halo exchange inside
    the timed region.  Strong scaling (fixed total image).  The K steps are
    captured in one CUDA graph (kernels + NCCL send/recv) when every rank's
    capture succeeds, else timed eagerly (the line says which)."""
    import torch
    import torch.distributed as dist

    import paper_2203_10670_b200 as fc
    from paper_2203_10670_b200.dist import StripRunner

    pl = make_plan(fc, cfg)
    esz = {"float32": 4, "float16": 2, "bfloat16": 2}[cfg.dtype]
    halo = args.halo
    sr = StripRunner(pl, rank, world, transport=halo)
    lay = sr.lay
    x_host = synth.make_input(cfg, rows=(lay.own0, lay.own1))
    x_own = x_host.to(dev)
    stream = torch.cuda.Stream(dev)
    R = 3  # rotating local/output buffers (each >= 4 x 32768 x 4 KB)
    outs = [sr.alloc_out(1, x_own.dtype, dev) for _ in range(R)]
    if halo == "peer":  # one symmetric-memory strip per rank; neighbours read it in place
        sr.setup_peer(1, x_own.dtype, dev).copy_(x_own)
        locs = [None] * R

        def run(k):
            sr.run_peer(outs[k % R])
    else:
        locs = [sr.alloc_local(1, x_own.dtype, dev) for _ in range(R)]
        for buf in locs:
            sr.own_view(buf).copy_(x_own)

        def run(k):
            sr.run(locs[k % R], outs[k % R])
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(physical_gpu_index(int(os.environ.get("LOCAL_RANK", "0"))))
    sampler.start()
    t0 = time.time()
    k = 0
    with torch.cuda.stream(stream):
        while time.time() - t0 < args.soak_s:
            run(k)
            k += 1
            if k % 20 == 0:
                torch.cuda.synchronize(dev)
        for w in range(args.warmup):
            run(w)
    torch.cuda.synchronize(dev)
    # one CUDA graph of the K steps (every rank must capture, or none replays)
    graph, how = None, "eager"
    n_launch0 = fc.kernel_launches()
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for st in range(args.steps):
                run(st)
        graph, how = g, "cuda_graph"
    except Exception as e:  # noqa: BLE001 -- reported in the line, timed eagerly instead
        how = f"eager (graph capture failed: {type(e).__name__}: {str(e)[:120]})"
        torch.cuda.synchronize(dev)
    n_launches = fc.kernel_launches() - n_launch0
    if world > 1:
        ok = torch.tensor([1.0 if graph is not None else 0.0], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() < 1.0 and graph is not None:
            graph, how = None, "eager (another rank's graph capture failed)"
    if graph is not None:
        with torch.cuda.stream(stream):
            graph.replay()  # upload / warm-up
    else:
        n_launch0 = fc.kernel_launches()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            for st in range(args.steps):
                run(st)
        e1.record(stream)
    if graph is None:
        n_launches = fc.kernel_launches() - n_launch0
    torch.cuda.synchronize(dev)
    t1 = time.time()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clocks = sampler.summary(t0, t1)
    sampler.stop()
    outputs = pl.Ho * pl.Wo
    total_bytes = pl.compulsory_bytes(1)
    ms_step = ms / args.steps
    peak, kind = peaks()
    # per-rank algorithmic bytes: own output rows + own + halo input rows
    rank_bytes = ((lay.out1 - lay.out0) * pl.Wo + (lay.loc1 - lay.loc0) * pl.W) * esz
    achieved = rank_bytes / (ms_step * 1e-3) / 1e9

    # e2e: every step copies this rank's strip in from pinned memory, runs the
    # strip step (exchange + kernels) and reads its output rows back
    e2e = None
    if not args.no_e2e:
        pin_in = x_host.pin_memory()
        pin_out = torch.empty(outs[0].shape, dtype=outs[0].dtype).pin_memory()
        tgt = sr.local if halo == "peer" else sr.own_view(locs[0])
        steps = max(1, min(args.steps, 20))
        with torch.cuda.stream(stream):
            for k in range(2):
                tgt.copy_(pin_in, non_blocking=True)
                run(0)
                pin_out.copy_(outs[0], non_blocking=True)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            f0.record(stream)
            for k in range(steps):
                tgt.copy_(pin_in, non_blocking=True)
                run(0)
                pin_out.copy_(outs[0], non_blocking=True)
            f1.record(stream)
        torch.cuda.synchronize(dev)
        ems = f0.elapsed_time(f1)
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": outputs * steps / (ems * 1e-3) / 1e6, "unit": "Mpix/s",
               "h2d_bytes_per_step": pin_in.numel() * esz, "d2h_bytes_per_step": pin_out.numel() * esz,
               "steps": steps, "ms_per_step": ems / steps,
               "path": "per rank: pinned own strip -> HBM -> strip step (halo exchange + fcfs_run_rows) -> "
                       "pinned own output rows (bytes per rank)"}

    line = {"metric": METRIC, "value": outputs * args.steps / (ms * 1e-3) / 1e6, "unit": "Mpix/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": DTYPE_TAG[cfg.dtype],
            "data": "synthetic",
            "config": {"workload": "C5", "shape": [1, 1, cfg.H, cfg.W], "factor": f"{cfg.p}/{cfg.q}",
                       "mode": cfg.mode, "pad": cfg.pad, "out": [pl.Ho, pl.Wo],
                       "parallelism": (f"row strips x{world}, NCCL halo send/recv, interior overlapped" if halo == "nccl"
                                       else f"row strips x{world}, halo rows read in-kernel from the neighbours' "
                                            "symmetric-memory strips (peer pointers), device barriers per step"),
                       "rank0_rows": {"own_in": [lay.own0, lay.own1], "out": [lay.out0, lay.out1]},
                       "l2": "working set per rank > L2; 3 rotating buffer sets",
                       "timing": how},
            "achieved_GBps_step": total_bytes / (ms_step * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None,
                         "peak_source": f"{kind} MEASURED_PEAKS.json hbm_gbs",
                         "note": "rank-0 bytes (own output rows + own and halo input rows) / max-over-ranks step "
                                 "time (exchange included)"},
            "gpu_launches": n_launches, "clocks": clocks, "provenance": provenance()}
    if e2e is not None:
        line["e2e"] = e2e
    if rank == 0 and not args.no_cpu_baseline:
        def gpu_result(name, what):
            assert what[0] == "rows" and lay.out0 <= what[1] and what[2] <= lay.out1
            rng = float((x_own.max() - x_own.min()).item())  # rank 0's rows: the sample reads only those
            return outs[0][:, :, what[1] - lay.out0:what[2] - lay.out0].cpu(), rng
        line["cpu_baseline"] = cpu_baseline([cfg], gpu_result=gpu_result)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_e2e(launches, args, dev, stream, world, dist, fc=None, groups=None, total_outputs=None):
    """Same metric through the public host-buffer call (fcfs_run_host): every step
    copies its inputs H2D from pinned memory, runs, and reads the outputs D2H.
    Consecutive steps alternate between two streams with their own device and
    pinned output buffers, so one step's D2H overlaps the next step's H2D (the
    two copy engines), as a pipelined caller would use the API."""
    import torch
    pin_in = {}
    for L in launches:
        if L["key"] not in pin_in:
            pin_in[L["key"]] = L["x_host"].pin_memory()
        L["pin_outs"] = [torch.empty(L["outs"][0].shape, dtype=L["outs"][0].dtype).pin_memory() for _ in range(2)]
        L["pin_out"] = L["pin_outs"][0]
    dins = [{k: torch.empty(v.shape, dtype=v.dtype, device=dev) for k, v in pin_in.items()} for _ in range(2)]
    # device outputs of their own per stream (never shared with the other stream)
    douts = [[torch.empty(L["outs"][0].shape, dtype=L["outs"][0].dtype, device=dev) for L in launches]
             for _ in range(2)]
    for li, L in enumerate(launches):
        L["e2e_outs"] = [douts[0][li], douts[1][li]]
    pin_g = {L["key"]: L["g_host"].pin_memory() for L in launches if L["cfg"].wgrad}
    gdevs = [{k: torch.empty(v.shape, dtype=v.dtype, device=dev) for k, v in pin_g.items()} for _ in range(2)]
    streams = [stream, torch.cuda.Stream(dev)]
    # a workload of several forward launches over one batch (C2, C4: two factors)
    # copies the batch in once per step and runs every launch on it (run_batch
    # where the launches share a kernel launch); single launches use the
    # one-call host path
    batched = (groups is not None and fc is not None and len(launches) > 1 and
               not any(L["cfg"].backward or L["cfg"].wgrad for L in launches))
    if batched:
        h2d = sum(v.numel() * v.element_size() for v in pin_in.values())
    else:
        h2d = sum(pin_in[L["key"]].numel() * pin_in[L["key"]].element_size() for L in launches) + \
            sum(v.numel() * v.element_size() for v in pin_g.values())
    d2h = sum(L["pin_out"].numel() * L["pin_out"].element_size() for L in launches)

    def step(k):
        i = k % 2
        st, din, gdev = streams[i], dins[i], gdevs[i]
        if batched:  # copy the batch in once, one fcfs_run_batch launch, copy every output back
            with torch.cuda.stream(st):
                for key, v in pin_in.items():
                    din[key].copy_(v, non_blocking=True)
                for grp in groups:
                    if len(grp) > 1:
                        fc.run_batch([(launches[j]["plan"], din[launches[j]["key"]], launches[j]["e2e_outs"][i])
                                      for j in grp], stream=st)
                    else:
                        L = launches[grp[0]]
                        L["plan"].run(din[L["key"]], out=L["e2e_outs"][i], stream=st)
                for L in launches:
                    L["pin_outs"][i].copy_(L["e2e_outs"][i], non_blocking=True)
            return
        for L in launches:
            out_d, out_h = L["e2e_outs"][i], L["pin_outs"][i]
            if L["cfg"].backward:  # public API: copy in, Plan.run_adjoint, copy out (all on the stream)
                with torch.cuda.stream(st):
                    din[L["key"]].copy_(pin_in[L["key"]], non_blocking=True)
                    L["plan"].run_adjoint(din[L["key"]], out=out_d, stream=st)
                    out_h.copy_(out_d, non_blocking=True)
            elif L["cfg"].wgrad:  # copy x and grad_out in, Plan.run_weight_grad, copy grad_w out
                with torch.cuda.stream(st):
                    din[L["key"]].copy_(pin_in[L["key"]], non_blocking=True)
                    gdev[L["key"]].copy_(pin_g[L["key"]], non_blocking=True)
                    L["plan"].run_weight_grad(din[L["key"]], gdev[L["key"]], out=out_d, stream=st)
                    out_h.copy_(out_d, non_blocking=True)
            else:
                L["plan"].run_host(pin_in[L["key"]], out_h, din[L["key"]], out_d, stream=st)

    for k in range(max(2, args.warmup)):
        step(k)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    steps = max(1, min(args.steps, 50))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    streams[1].wait_event(e0)
    for k in range(steps):
        step(k)
    done1 = torch.cuda.Event()
    done1.record(streams[1])
    stream.wait_event(done1)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    outputs = total_outputs if total_outputs is not None else world * sum(L["outputs"] for L in launches)
    return {"value": outputs * steps / (ms * 1e-3) / 1e6, "unit": "Mpix/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps, "ms_per_step": ms / steps,
            "path": ("pinned batch -> HBM once -> every factor's launch (fcfs_run_batch / fcfs_run) -> pinned outputs"
                     if batched else
                     "pinned grad_out -> HBM -> fcfs_run_adjoint -> pinned grad_in" if launches[0]["cfg"].backward else
                     "pinned x, grad_out -> HBM -> fcfs_run_weight_grad -> pinned grad_w" if launches[0]["cfg"].wgrad
                     else "fcfs_run_host (pinned host -> HBM -> kernel -> pinned host)") +
                    "; steps alternate between two streams (D2H of one overlaps H2D of the next)"}


if __name__ == "__main__":
    sys.exit(main())
