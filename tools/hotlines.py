"""Executed instructions and stall samples per source line of an ncu report (developer tool).

    python tools/hotlines.py report.ncu-rep [--top 25]
"""
import argparse
import collections
import importlib.util
import os

spec = importlib.util.spec_from_file_location("ns", os.path.join(os.path.dirname(__file__), "ncu_summary.py"))
ns = importlib.util.module_from_spec(spec)
spec.loader.exec_module(ns)
ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=25)
a = ap.parse_args()
rows = ns.ncu_csv(["-i", a.rep, "--page", "source", "--print-source", "cuda,sass"])
cur_file, hdr, cur_line = None, None, None
inst, stall, src = collections.Counter(), collections.Counter(), {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0] != "":
        cur_line = (cur_file, int(r[0]))
        src[cur_line] = r[1].strip()
        continue
    try:
        inst[cur_line] += int(r[7] or 0)
        stall[cur_line] += int(r[4] or 0)
    except ValueError:
        pass
I, S = sum(inst.values()) or 1, sum(stall.values()) or 1
print(f"total executed warp instructions {I / 1e6:.1f} M")
for k, v in inst.most_common(a.top):
    print(f"{100 * v / I:5.1f}% {v / 1e6:7.1f}M  stall {100 * stall[k] / S:5.1f}%  {k[0]}:{k[1]}  {src.get(k, '')[:90]}")
