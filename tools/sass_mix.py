"""Executed-instruction mix by SASS opcode from an ncu report (developer tool).

    python tools/sass_mix.py report.ncu-rep [--kernel N] [--top 40]
"""
import argparse
import collections
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--stalls", action="store_true", help="also list the top stall instructions")
args = ap.parse_args()
out = subprocess.run(["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name"')
for blk in blocks[1:]:
    lines = blk.splitlines()
    name = lines[0].strip(",")
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    ia, isrc, iex, ist = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index(
        "Warp Stall Sampling (All Samples)")
    mix = collections.Counter()
    tot = 0
    ins = []
    for r in rows[1:]:
        if len(r) <= iex:
            continue
        try:
            n = int(float(r[iex]))
            s = int(float(r[ist]))
        except ValueError:
            continue
        op = r[isrc].strip().split()
        if not op:
            continue
        o = op[0]
        if o.startswith("@"):
            o = op[1] if len(op) > 1 else o
        mix[o.split(".")[0] if not o.startswith(("FFMA2", "FMUL2")) else o] += n
        tot += n
        ins.append((s, n, r[ia], r[isrc].strip()))
    print(name, "total warp inst", tot)
    for o, n in mix.most_common(args.top):
        print(f"  {o:14s} {n:12d} {100 * n / tot:6.2f}%")
    if args.stalls:
        ins.sort(reverse=True)
        for s, n, a, src in ins[:30]:
            print(f"  stall {s:7d} exec {n:9d} {src}")
