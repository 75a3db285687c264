#!/usr/bin/env python
"""Summarise ncu output for profiles/.

  tools/ncu_summary.py launches <launches.csv>            per-kernel share of the step (gpu__time_duration)
  tools/ncu_summary.py report <report.ncu-rep>             key metrics per captured launch (ncu --set full)
"""
import collections
import csv
import io
import re
import subprocess
import sys


def _short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("gsc::", "").replace("void ", "")
    return name


def launches(path):
    rows = []
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    rd = csv.DictReader(io.StringIO("".join(lines)))
    for r in rd:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((_short(r["Kernel Name"]), float(r["Metric Value"]) / 1e3))  # us
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for k, us in rows:
        tot[k] += us
        cnt[k] += 1
    T = sum(tot.values())
    out = ["| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        out.append(f"| {k} | {cnt[k]} | {v:.0f} | {v / cnt[k]:.1f} | {100 * v / T:.1f}% |")
    out.append(f"| **all** | {len(rows)} | {T:.0f} | | 100% |")
    return "\n".join(out)


WANT = [
    ("Duration", "Duration"), ("DRAM Throughput", "DRAM %"), ("Memory Throughput", "Mem"),
    ("Compute (SM) Throughput", "SM %"), ("Issue Slots Busy", "issue %"), ("Executed Ipc Active", "IPC"),
    ("Achieved Occupancy", "occ %"), ("Registers Per Thread", "regs"), ("L2 Hit Rate", "L2 hit %"),
    ("Warp Cycles Per Issued Instruction", "cyc/inst"),
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed.sum",
       "smsp__inst_executed_pipe_fma.sum", "smsp__inst_executed_pipe_alu.sum", "smsp__inst_executed_pipe_lsu.sum",
       "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def report(path):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rd = list(csv.reader(io.StringIO(det)))
    hdr = rd[0]
    ii, ki, mi, vi, ui = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    per = collections.OrderedDict()
    for r in rd[1:]:
        key = (r[ii], _short(r[ki]))
        per.setdefault(key, {})
        for m, short in WANT:
            if r[mi] == m and short not in per[key]:
                per[key][short] = f"{r[vi]} {r[ui]}".strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    rh = rr[0]
    cols = {m: rh.index(m) for m in RAW if m in rh}
    units = rr[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rid, rk = rh.index("ID"), rh.index("Kernel Name")
    for r in rr[2:]:
        key = (r[rid], _short(r[rk]))
        if key not in per:
            continue
        for m, c in cols.items():
            v = r[c]
            if units[c] in scale:
                v = str(float(v.replace(",", "")) * scale[units[c]])
            per[key][m] = v
    heads = [s for _, s in WANT] + ["dram read+write"] + [m for m in RAW[2:] if m in cols]
    out = ["| id | kernel | " + " | ".join(heads) + " |", "|" + "---|" * (len(heads) + 2)]
    for (i, k), d in per.items():
        try:
            traffic = float(d.get("dram__bytes_read.sum", "nan").replace(",", "")) + \
                float(d.get("dram__bytes_write.sum", "nan").replace(",", ""))
            d["dram read+write"] = f"{traffic / 1e6:.1f} MB"
        except ValueError:
            d["dram read+write"] = "n/a"
        out.append(f"| {i} | {k} | " + " | ".join(d.get(h, "") for h in heads) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(launches(path) if mode == "launches" else report(path))
