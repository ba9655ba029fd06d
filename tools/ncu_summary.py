"""Summarise ncu reports into profiles/ (developer tool; runs without a GPU).

    python tools/ncu_summary.py <report.ncu-rep> --out profiles/r01_C3_fused.md [--traffic-key C3]
    python tools/ncu_summary.py --launches gpurun_out/launches.csv --out profiles/r01_launches.md

Writes the key metrics of every profiled kernel (duration, DRAM bytes, achieved
DRAM bandwidth, instruction mix, stall reasons, shared-memory wavefronts) and
the hottest source lines; with --traffic-key it also records the kernel's DRAM
read+write bytes per launch in profiles/traffic.json (bench.py's roofline
"traffic" field).
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read (MB)"),
    ("dram__bytes_write.sum", "DRAM write (MB)"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% of peak)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM, active)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy (%)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput (%)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "shared-memory wavefronts (% of peak)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem store bank conflicts"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy (%)"),
]
STALLS = ["barrier", "long_scoreboard", "short_scoreboard", "wait", "math_pipe_throttle", "no_instruction",
          "mio_throttle", "lg_throttle", "not_selected", "branch_resolving", "sleeping", "membar", "dispatch_stall"]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def raw_rows(rep):
    rows = ncu_csv(["-i", rep, "--page", "raw"])
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def fnum(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return float("nan")


def hot_lines(rep, top=15):
    rows = ncu_csv(["-i", rep, "--page", "source", "--print-source", "cuda,sass"])
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
    S = sum(stall.values()) or 1
    I = sum(inst.values()) or 1
    return [(k, 100 * inst[k] / I, 100 * stall[k] / S, src.get(k, "")) for k, _ in stall.most_common(top)]


def summarise(rep, out, traffic_key=None, title=None, traffic_match=None):
    kernels, units = raw_rows(rep)
    lines = [f"# {title or os.path.basename(rep)}", "", f"Source report: `{os.path.basename(rep)}` "
             "(`ncu --set full --clock-control none --import-source on`, one launch).", ""]
    traffic = None
    per_name = {}  # a launch group of several kernels (C3B: fused adjoint + bands): their sum
    for d in kernels:
        name = d.get("Kernel Name", "?")
        lines += [f"## `{name}`", "", "| metric | value |", "|---|---|"]
        for key, label in METRICS:
            if key in d:
                v = fnum(d[key])
                u = units.get(key, "")
                if key.startswith("dram__bytes") and u.lower().startswith("mbyte"):
                    pass
                lines.append(f"| {label} | {d[key]} {u} |")
        dur = fnum(d.get("gpu__time_duration.sum"))
        rd = fnum(d.get("dram__bytes_read.sum"))
        wr = fnum(d.get("dram__bytes_write.sum"))
        scale = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}
        ru = scale.get(units.get("dram__bytes_read.sum", "byte").lower(), 1)
        wu = scale.get(units.get("dram__bytes_write.sum", "byte").lower(), 1)
        du = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
              "s": 1.0}[units.get("gpu__time_duration.sum", "").strip().lower()]
        tot = rd * ru + wr * wu
        if traffic_match is None or traffic_match in name:  # (C4: only the dominant launch's kernel)
            per_name.setdefault(name, tot)
        traffic = sum(per_name.values()) if per_name else None
        lines.append(f"| DRAM read+write per launch | {tot / 1e6:.3f} MB |")
        if dur == dur and dur > 0:
            lines.append(f"| achieved DRAM bandwidth (under ncu, cold) | {tot / (dur * du) / 1e9:.1f} GB/s |")
        lines += ["", "Stall reasons (warps per issue-active cycle):", "", "| reason | ratio |", "|---|---|"]
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in d and fnum(d[k]) > 0.01:
                lines.append(f"| {s} | {fnum(d[k]):.3f} |")
        lines.append("")
    try:
        hl = hot_lines(rep)
        lines += ["Hottest source lines (share of stall samples / of executed instructions):", "",
                  "| stall % | inst % | line | source |", "|---|---|---|---|"]
        for (f, ln), ip, sp, s in hl:
            lines.append(f"| {sp:.1f} | {ip:.1f} | {f}:{ln} | `{s[:90].replace('|', '/')}` |")
    except Exception as e:  # source page needs -lineinfo
        lines.append(f"(source page unavailable: {e})")
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    open(out, "w").write("\n".join(lines) + "\n")
    if traffic_key and traffic is not None:
        path = os.path.join(ROOT, "profiles", "traffic.json")
        tj = json.load(open(path)) if os.path.exists(path) else {}
        tj[traffic_key] = int(traffic)
        json.dump(tj, open(path, "w"), indent=1, sort_keys=True)


def launches(csv_path, out):
    rows = list(csv.reader(open(csv_path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    recs = [dict(zip(hdr, r)) for r in rows[start + 1:] if len(r) == len(hdr)]
    per = collections.defaultdict(list)
    for r in recs:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            per[r["Kernel Name"]].append(fnum(r["Metric Value"]))
    total = sum(sum(v) for v in per.values()) or 1
    lines = [f"# Launch list: `{os.path.basename(csv_path)}`", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` over the bench command "
             "(cold-cache, serialised launches: compare shares, not absolutes).", "",
             "| kernel | launches | mean | share of time |", "|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k[:100]}` | {len(v)} | {sum(v) / len(v):.2f} | {100 * sum(v) / total:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("report", nargs="?")
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic-key")
    ap.add_argument("--title")
    ap.add_argument("--traffic-match", help="only kernels whose name contains this count toward the traffic key")
    ap.add_argument("--launches")
    a = ap.parse_args()
    if a.launches:
        launches(a.launches, a.out)
    else:
        summarise(a.report, a.out, a.traffic_key, a.title, a.traffic_match)
    print(a.out)
