"""DRAM traffic of the smoother launches of the TIMED steps of bench.py.

The capture (on the GPU box) replays the whole application with caches left
as the program leaves them (not flushed per kernel), so the L2 state each
colour launch sees is the one of the real step (L2 flushed before the step,
the earlier colours' x / b lines resident):

  ncu --replay-mode application --cache-control none --clock-control none \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      -k regex:vp_ --csv --log-file OUT.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu --no-sweep

python tools/ncu_step_traffic.py OUT.csv KEY --skip 24 --per-step 8 --steps 3

KEY is bench.py's ncu_summary key (d{dim}k{k}L{L}{dtype}{variant}); --skip the
warm-up launches before the timed region. Writes dram_bytes_per_step (mean
over the timed steps) into profiles/ncu_summary.json.
"""

import argparse
import csv
import io
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def read_launches(path):
    text = open(path).read()
    i = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[i:])))
    hdr = rows[0]
    col = {h: j for j, h in enumerate(hdr)}
    per = {}
    order = []
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        lid = int(r[col["ID"]])
        name = r[col["Metric Name"]]
        unit = r[col["Metric Unit"]]
        val = float(r[col["Metric Value"]].replace(",", "")) * UNIT.get(unit, 1.0)
        if lid not in per:
            per[lid] = {"kernel": r[col["Kernel Name"]]}
            order.append(lid)
        per[lid][name] = val
    return [per[i] for i in order]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("key")
    ap.add_argument("--skip", type=int, required=True)
    ap.add_argument("--per-step", type=int, default=8)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--source", default=None)
    a = ap.parse_args()
    L = read_launches(a.csv)
    steps = []
    for s in range(a.steps):
        ls = L[a.skip + s * a.per_step: a.skip + (s + 1) * a.per_step]
        assert len(ls) == a.per_step, (len(L), a.skip, s)
        steps.append({"dram_bytes": sum(x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in ls),
                      "dram_read": sum(x["dram__bytes_read.sum"] for x in ls),
                      "dram_write": sum(x["dram__bytes_write.sum"] for x in ls),
                      "launch_bytes": [x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in ls],
                      "kernels": sorted({x["kernel"].split("(")[0] for x in ls})})
    mean = sum(s["dram_bytes"] for s in steps) / len(steps)
    summ = json.load(open(SUMMARY)) if os.path.exists(SUMMARY) else {}
    ent = summ.get(a.key, {})
    ent["dram_bytes_per_step"] = mean
    ent["dram_bytes_per_launch_in_step"] = steps[0]["launch_bytes"]
    ent["note"] = ("DRAM read+write of the timed steps' smoother launches, ncu --replay-mode application "
                   "--cache-control none (L2 state of the real step); per launch = per step / launches")
    ent["step_source"] = a.source or os.path.relpath(a.csv, ROOT)
    summ[a.key] = ent
    json.dump(summ, open(SUMMARY, "w"), indent=1, sort_keys=True)
    for i, s in enumerate(steps):
        print(f"step {i}: DRAM {s['dram_bytes'] / 1e6:.1f} MB (read {s['dram_read'] / 1e6:.1f}, "
              f"write {s['dram_write'] / 1e6:.1f}); kernels {s['kernels']}")
    print(f"mean {mean / 1e6:.1f} MB per step -> {SUMMARY}")


if __name__ == "__main__":
    main()
