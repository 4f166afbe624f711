"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ launch__grid_size])
per kernel launch, in order: python tools/debug/ncu_kernels.py file.csv [filter]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
flt = sys.argv[2] if len(sys.argv) > 2 else ""
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d, order = {}, []
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    if r[idi] not in d:
        d[r[idi]] = {"name": r[ki]}
        order.append(r[idi])
    d[r[idi]][r[mi]] = r[vi]
tot = 0.0
for kid in order:
    e = d[kid]
    t = float(e["gpu__time_duration.sum"].replace(",", "")) / 1000
    tot += t
    nm = e["name"].split("(")[0].replace("void pmgb::", "")[:58]
    if flt in nm:
        print(f"{kid:>4} {nm:58s} grid={e.get('launch__grid_size', '?'):>8} {t:8.2f} us")
print(f"total {tot:.1f} us over {len(order)} launches")
