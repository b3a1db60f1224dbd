"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`) by
kernel: launches, total / mean duration and share of the summed kernel time.

  python scripts/launch_breakdown.py gpurun_out/launches.csv [--top 25]
"""
import argparse
import csv
import io
import re
from collections import defaultdict


def load(path):
    text = open(path, errors="replace").read()
    start = text.find('"ID"')
    rows = csv.DictReader(io.StringIO(text[start:]))
    out = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                 "nsecond": 1e-3, "second": 1e6}.get(unit, 1e-3)
        out.append((r["Kernel Name"], v * scale))
    return out


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name[:90]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    rows = load(a.csv)
    agg = defaultdict(lambda: [0, 0.0])
    for n, us in rows:
        k = short(n)
        agg[k][0] += 1
        agg[k][1] += us
    total = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, {total / 1e3:.2f} ms summed kernel time (serialised, cold)")
    print(f"{'kernel':90s} {'n':>6s} {'total ms':>9s} {'mean us':>9s} {'share':>6s}")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:a.top]:
        print(f"{k:90s} {n:6d} {us / 1e3:9.2f} {us / n:9.1f} {us / total:6.1%}")


if __name__ == "__main__":
    main()
