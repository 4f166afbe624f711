"""Executed-instruction histogram (by opcode) from an ncu source page, with
an optional address window. python tools/sass_hist.py REP [lo hi]"""
import csv, io, subprocess, sys
from collections import defaultdict
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]; ix = {n: i for i, n in enumerate(h)}
hist = defaultdict(float); tot = 0
seq = []
for r in rows[2:]:
    if len(r) != len(h): continue
    n = float(r[ix["Instructions Executed"]].replace(",", "") or 0)
    src = r[ix["Source"]].split()
    if not src: continue
    op = src[1] if src[0].startswith("@") else src[0]
    seq.append((r[ix["Address"]], op, n))
    hist[op.split(".")[0]] += n; tot += n
print(f"total warp-instructions {tot:.0f}")
for k, v in sorted(hist.items(), key=lambda x: -x[1])[:25]:
    print(f"  {k:10s} {v:12.0f} {100*v/tot:5.1f}%")
if len(sys.argv) > 2:
    for a, op, n in seq:
        print(a, op, n)
