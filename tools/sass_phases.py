"""Warp-stall samples and executed instructions per barrier-delimited phase
of a kernel (ncu source page, SASS). python tools/sass_phases.py REP [launch]"""
import csv, io, subprocess, sys
from collections import defaultdict
args = ["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"]
if len(sys.argv) > 2:
    args += ["--launch-skip", sys.argv[2], "--launch-count", "1"]
raw = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = [i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r][0]
h = rows[hi]; ix = {n: i for i, n in enumerate(h)}
stall_cols = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
phase = 0; acc = defaultdict(lambda: defaultdict(float)); names = {}
end = [i for i, r in enumerate(rows) if i > hi and r and r[0] == "Kernel Name"]
stop = end[0] if end else len(rows)
for r in rows[hi + 1:stop]:
    if len(r) != len(h): continue
    src = r[ix["Source"]]
    def f(n):
        try: return float(r[ix[n]].replace(",", "") or 0)
        except ValueError: return 0.0
    a = acc[phase]
    a["samples"] += f("Warp Stall Sampling (All Samples)")
    a["inst"] += f("Instructions Executed")
    for n in stall_cols: a[n] += f(n)
    if "BAR.SYNC" in src or "BAR.RED" in src:
        phase += 1
tot = sum(a["samples"] for a in acc.values())
for p, a in sorted(acc.items()):
    top = sorted(((a[n], n[6:]) for n in stall_cols), reverse=True)[:4]
    print(f"phase {p}: {100*a['samples']/tot:5.1f}% samples, {a['inst']:10.0f} warp-inst; " +
          ", ".join(f"{n}={100*v/max(a['samples'],1):.0f}%" for v, n in top))
