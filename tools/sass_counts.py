#!/usr/bin/env python
"""Per-SASS-instruction executed counts of one kernel in an ncu report
(`--import-source on`), in address order, with the share of all warp-level
instructions: where the issue slots go.

  tools/sass_counts.py <report.ncu-rep> <kernel-name-substring> [min_share_percent]
"""
import csv
import io
import subprocess
import sys


def main(rep, kern, thr=0.0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern,
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = {k: i for i, k in enumerate(rows[0])}
    recs = []
    for r in rows[1:]:
        try:
            n = int(r[h["Instructions Executed"]] or 0)
        except (ValueError, IndexError):
            continue
        recs.append((r[h["Address"]], r[h["Source"]], n, r[h["Avg. Threads Executed"]]))
    tot = sum(n for _, _, n, _ in recs)
    print(f"total warp instructions {tot:,}")
    for a, s, n, t in recs:
        if n * 100.0 / tot >= thr:
            print(f"{a[-5:]} {n:>12,} {n * 100.0 / tot:5.2f}% thr={t:>5} {s.strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else 0.0)
