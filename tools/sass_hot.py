import csv, sys, collections
# usage: python tools_sass_hot.py report kernel [n]
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
import subprocess
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern, "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
idx = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
lines = []
for r in rows[1:]:
    try:
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    lines.append((s, r[idx["Address"]], r[idx["Source"]], {c: r[idx[c]] for c in stall_cols}))
    for c in stall_cols:
        try:
            tot[c] += int(r[idx[c]] or 0)
        except ValueError:
            pass
S = sum(l[0] for l in lines)
print("total samples", S)
print("stalls:", ", ".join(f"{k[6:]}={v*100/S:.1f}%" for k, v in tot.most_common(8)))
for s, a, src, st in sorted(lines, key=lambda l: -l[0])[:n]:
    top = sorted(((int(v or 0), k[6:]) for k, v in st.items() if v and v != '0'), reverse=True)[:3]
    print(f"{s*100/S:5.1f}% {a} {src[:60]:60s} {top}")
