"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv`)
into the markdown table kept under profiles/ (kernel, launches, mean ns, share)."""
import csv
import io
import sys
from collections import OrderedDict


def summarise(path: str) -> str:
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"]
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + float(r["Metric Value"].replace(",", "")))
    total = sum(t for _, t in agg.values()) or 1.0
    out = [f"# Launch list: `{path.split('/')[-1]}`", "",
           "`ncu --metrics gpu__time_duration.sum --clock-control none` over the bench command "
           "(cold-cache, serialised launches: compare shares, not absolutes).", "",
           "| kernel | launches | mean | share of time |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k[:100]}` | {n} | {t / n:.2f} | {100 * t / total:.1f}% |")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    src, dst = sys.argv[1], sys.argv[2]
    open(dst, "w").write(summarise(src))
