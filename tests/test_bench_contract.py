"""bench.py contract checks that run without a GPU: the reference arm (the
oracle timed on the host) prints one JSON line with the keys the
driver reads, on the same metric / unit / config as the GPU arm."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1", "--workload", "C1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "Mpix/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"] == "C1"


def test_workloads_are_known_configs():
    sys.path.insert(0, ROOT)
    import synth
    for name, launches in synth.WORKLOADS.items():
        for l in launches:
            assert l in synth.CONFIGS, (name, l)


def test_oracle_legs_of_the_backward_workloads():
    """The cpu_baseline / --impl reference legs of C3B and C3W time the oracle's
    adjoint and weight gradient (not the forward) on a sample of whole planes."""
    sys.path.insert(0, ROOT)
    import bench
    import synth
    for name, what in (("C3B", "adjoint"), ("C3W", "weight gradient")):
        outs, secs, desc = bench.oracle_sample_run([synth.CONFIGS[name]], 1)
        assert outs == synth.CONFIGS[name].C * 213 * 213 and secs > 0 and what in desc, (name, desc)


def test_config1_oracle_single_thread_well_under_a_second():
    """BASELINE.json config 0: 'CPU oracle runs in well under a second' -- the
    staged oracle on C1a (48x64 bilinear 3/2) and C1b (1D 101 nearest 2/3) on
    one thread (report a 1-thread time for C1a/C1b)."""
    import time
    sys.path.insert(0, ROOT)
    import oracle
    import synth
    for name in ("C1a", "C1b"):
        c = synth.CONFIGS[name]
        x = synth.make_values(c)
        t0 = time.perf_counter()
        oracle.staged(x, c.p, c.q, c.mode, c.pad, floor_extent=c.floor_extent, is1d=c.is1d, nthreads=1)
        dt = time.perf_counter() - t0
        assert dt < 0.5, (name, dt)
