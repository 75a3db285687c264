#!/usr/bin/env python
"""Stall-sampling hotspots of one kernel launch in an ncu report (--import-source on).

  tools/ncu_stalls.py <report.ncu-rep> <launch index in the report> [n lines]
"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, idx, n=20):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    print(lines[0][:160])
    start = [i for i, l in enumerate(lines) if l.startswith('"Address"')][0]
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    h = {k: i for i, k in enumerate(rows[0])}
    stall_cols = [k for k in rows[0] if k.startswith("stall_") and "Not Issued" not in k]
    tot, recs = collections.Counter(), []
    for r in rows[1:]:
        try:
            s = int(r[h["Warp Stall Sampling (All Samples)"]] or 0)
            ex = int(r[h["Instructions Executed"]] or 0)
        except (ValueError, IndexError):
            continue
        recs.append((s, ex, r[h["Address"]], r[h["Source"]], {c: r[h[c]] for c in stall_cols}))
        for c in stall_cols:
            try:
                tot[c] += int(r[h[c]] or 0)
            except ValueError:
                pass
    S = sum(x[0] for x in recs) or 1
    E = sum(x[1] for x in recs) or 1
    print(f"samples {S}, warp instructions {E:,}")
    print(", ".join(f"{k[6:]}={v * 100 / S:.1f}%" for k, v in tot.most_common(8)))
    for s, ex, a, src, st in sorted(recs, key=lambda x: -x[0])[:n]:
        top = sorted(((int(v or 0), k[6:]) for k, v in st.items() if v and v != '0'), reverse=True)[:3]
        print(f"{s * 100 / S:5.1f}% {a[-5:]} {src.strip()[:62]:62s} {top}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 20)
