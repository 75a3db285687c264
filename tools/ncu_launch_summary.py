#!/usr/bin/env python
"""Per-kernel launch count / total / mean duration from an ncu --csv gpu__time_duration.sum log.

  tools/ncu_launch_summary.py <launches.csv>
"""
import collections
import csv
import sys


def main(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.DictReader(lines[start:]))
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(r.get("Metric Unit", "usecond"), 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    tot = sum(a[1] for a in agg.values()) or 1.0
    print(f"{'kernel':60s} {'n':>5s} {'total us':>10s} {'mean us':>9s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:60]:60s} {n:5d} {t:10.1f} {t / n:9.2f} {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
