"""Per-SASS-instruction shared-memory wavefronts from an ncu source page.
python tools/sass_smem.py REP  -> instructions with shared wavefronts, and stall totals"""
import csv, io, subprocess, sys
from collections import defaultdict
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
ix = {n: i for i, n in enumerate(h)}
def f(r, n):
    try: return float(r[ix[n]].replace(",", ""))
    except (ValueError, KeyError): return 0.0
tot = defaultdict(float)
print("addr  source  exec  wavefronts  ideal")
for r in rows[2:]:
    if len(r) != len(h): continue
    wf = f(r, "L1 Wavefronts Shared"); ide = f(r, "L1 Wavefronts Shared Ideal")
    for n in h:
        if n.startswith("stall_") and "Not Issued" not in n:
            tot[n] += f(r, n)
    if wf > 0:
        print(f"{r[ix['Address']]:>6} {r[ix['Source']][:60]:60s} {f(r,'Instructions Executed'):9.0f} {wf:9.0f} {ide:9.0f} {wf/max(ide,1):5.2f}")
s = sum(tot.values())
print("stalls:", ", ".join(f"{k[6:]}={100*v/s:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:10]))
