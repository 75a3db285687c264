#!/usr/bin/env python
"""Per-CUDA-source-line instruction counts and stall samples of one kernel in an ncu report.

  tools/ncu_lines.py <report.ncu-rep> <kernel name> [top n]
"""
import csv
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern,
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout.splitlines()
    fname, hdr, rows = "?", None, []
    for rec in csv.reader(out):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname = rec[1].rsplit("/", 1)[-1]
            continue
        if rec[0] == "Line No":
            hdr = {h: i for i, h in enumerate(rec)}
            continue
        if hdr is None or rec[0] in ("Function Name",) or rec[2] != "-":
            continue
        try:
            samp = int(rec[hdr["Warp Stall Sampling (All Samples)"]] or 0)
            inst = int(rec[hdr["Instructions Executed"]] or 0)
        except (ValueError, IndexError):
            continue
        rows.append((fname, int(rec[0]), rec[1].strip(), samp, inst))
    S = sum(r[3] for r in rows) or 1
    I = sum(r[4] for r in rows) or 1
    print(f"samples {S}, warp instructions {I}")
    for f, ln, src, s, i in sorted(rows, key=lambda r: -r[4])[:n]:
        print(f"{100 * i / I:5.1f}% inst {100 * s / S:5.1f}% samp  {f}:{ln:<4d} {src[:90]}")


if __name__ == "__main__":
    main()
