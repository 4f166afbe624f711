"""Markdown tables from a bench.py JSON line: the C3 degree
sweep and the fused / naive / global comparator.

python tools/bench_tables.py profiles/r02/final4/bench.json
"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("| config | dtype | kernel | GDoF/s (step) | % FP peak (alg.) | % HBM (alg.) | V-cycle GDoF/s |")
print("|---|---|---|---|---|---|---|")
for s in d.get("sweep", []):
    print(f"| {s['dim']}D Q{s['degree']} L{s['level']} ({s['dofs']:.2e}) | {s['dtype']} | {s['kernel']} | "
          f"{s['value'] / 1e9:.1f} | {100 * s['fp_frac']:.1f} | {100 * s['hbm_frac']:.1f} | {s['vcycle_value'] / 1e9:.2f} |")
print()
print("| config | fused kernel | fused GDoF/s | naive GDoF/s | fused/naive | global GDoF/s | fused/global |")
print("|---|---|---|---|---|---|---|")
for c in d.get("comparator", []):
    print(f"| {c['dim']}D Q{c['degree']} L{c['level']} ({c['dofs']:.2e}) | {c['fused_kernel']} | {c['fused'] / 1e9:.2f} | "
          f"{c['naive'] / 1e9:.3f} | {c['speedup']:.1f}x | {c['global'] / 1e9:.2f} | {c['speedup_vs_global']:.2f}x |")
print()
r, rf = d["roofline"], d.get("roofline_fp", {})
print(f"headline {d['value'] / 1e9:.2f} GDoF/s, {d['ms_per_step']:.4f} ms/step, HBM frac {r['frac']:.3f}, "
      f"FP frac {rf.get('frac', float('nan')):.3f}, e2e {d['e2e']['value'] / 1e9:.2f} GDoF/s, "
      f"V-cycle {d['vcycle']['value'] / 1e9:.2f} GDoF/s ({d['vcycle']['ms']:.3f} ms), "
      f"cpu {d['cpu_baseline']['value'] / 1e6:.1f} MDoF/s on {d['cpu_baseline']['cores']} threads")
