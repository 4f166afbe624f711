"""Summarise `ncu --set full` captures of the smoother kernel.

python tools/ncu_summary.py OUT_DIR REP [REP ...]

For every .ncu-rep (one or more launches of vp_smooth_kernel, named
smooth_d{dim}k{k}L{L}{dtype}.ncu-rep) writes OUT_DIR/<name>.txt with the
counters the roofline argument rests on, and merges per-config totals into
profiles/ncu_summary.json (read by bench.py for roofline.traffic).
"""

import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "occupancy limit (registers)"),
    ("launch__occupancy_limit_shared_mem", "occupancy limit (smem)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 LSU wavefronts % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("memory_l1_wavefronts_shared_ideal", "smem wavefronts (ideal)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread-inst"),
    ("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "DMUL thread-inst"),
    ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "DADD thread-inst"),
    ("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "FFMA thread-inst"),
    ("smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "FMUL thread-inst"),
    ("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "FADD thread-inst"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
]

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
        "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9}


def launches(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m, _ in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[m] = v * UNIT.get(units[i], 1.0)
        out.append(d)
    return out


def main():
    outdir = sys.argv[1]
    os.makedirs(outdir, exist_ok=True)
    summary = json.load(open(SUMMARY)) if os.path.exists(SUMMARY) else {}
    for rep in sys.argv[2:]:
        name = os.path.basename(rep).replace(".ncu-rep", "")
        ls = launches(rep)
        lines = [f"# {name}: {len(ls)} launch(es) of {ls[0]['kernel'][:90] if ls else '?'}",
                 f"# source: ncu --set full --clock-control none ({os.path.basename(rep)})"]
        for j, d in enumerate(ls):
            lines.append(f"## launch {j}")
            for m, label in METRICS:
                if m in d:
                    v = d[m]
                    if m == "gpu__time_duration.sum":
                        s = f"{v * 1e6:.2f} us"
                    elif m.startswith("dram__bytes"):
                        s = f"{v / 1e6:.3f} MB"
                    elif abs(v) >= 1e5:
                        s = f"{v:.4g}"
                    else:
                        s = f"{v:.2f}"
                    lines.append(f"  {label:34s} {s:>14s}   ({m})")
            if "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum" in d and d.get("memory_l1_wavefronts_shared_ideal"):
                lines.append(f"  {'smem wavefronts / ideal':34s} "
                             f"{d['l1tex__data_pipe_lsu_wavefronts_mem_shared.sum'] / d['memory_l1_wavefronts_shared_ideal']:14.2f}")
        open(os.path.join(outdir, name + ".txt"), "w").write("\n".join(lines) + "\n")
        m = re.match(r"smooth_(d\dk\dL\d+f(?:32|64))(\w*)", name)
        if m and ls:
            key = m.group(1) + (m.group(2).lstrip("_") or "fused")
            dram = [d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in ls]
            summary[key] = {
                **{k: v for k, v in summary.get(key, {}).items() if k.startswith("dram_bytes_per_step") or k.endswith("_in_step") or k in ("note", "step_source")},
                "launches": len(ls),
                "dram_bytes_per_launch": dram,
                "duration_s_per_launch": [d.get("gpu__time_duration.sum") for d in ls],
                "dram_bytes_captured_total": sum(dram),
                "source": os.path.relpath(os.path.join(outdir, name + ".txt"), ROOT),
            }
        print("\n".join(lines[:40]))
    json.dump(summary, open(SUMMARY, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
