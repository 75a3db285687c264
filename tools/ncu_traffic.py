#!/usr/bin/env python
"""Write profiles/traffic.json: DRAM bytes (read + write) per launch of each
kernel in an `ncu --set full` report, for bench.py's roofline.traffic field.

  tools/ncu_traffic.py <report.ncu-rep> <label>
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rep, label):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, units = rr[0], rr[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    ir, iw, ik = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"), h.index("Kernel Name")
    out = {}
    for r in rr[2:]:
        name = re.sub(r"\(.*", "", r[ik]).replace("gsc::", "").replace("void ", "")
        name = re.sub(r"<.*>", "", name)
        b = float(r[ir].replace(",", "")) * scale[units[ir]] + float(r[iw].replace(",", "")) * scale[units[iw]]
        out.setdefault(name, []).append(b)
    res = {k: {"dram_bytes_per_launch": sum(v) / len(v), "launches": len(v), "source": label} for k, v in out.items()}
    path = os.path.join(ROOT, "profiles", "traffic.json")
    with open(path, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
