#!/usr/bin/env python
"""Benchmark of the vertex-patch smoother hot path (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--dim D --degree k --level L --dtype f64|f32 --variant fused]

One "step" = one colourised multiplicative vertex-patch smoothing step
(smooth<T>, /root/reference/proj/src/smoother.cpp:41-151) over the level's
synthetic x, b ~ U(-1,1). Default workload = BASELINE.json configs[1]
(3D Q2, 2^6 cells per direction, FP64). Prints ONE JSON line on rank 0.

Timing: W warm-up steps, then K steps each bracketed by CUDA events on the
launch stream, L2 flushed (write of a 256 MiB buffer) before every timed step
since the C2 vectors (2 x 16 MiB) fit in the 126 MB L2; barrier +
synchronize around the timed region, max over ranks. Clocks and throttle
reasons are sampled with NVML during the timed region.

Multi-GPU (torchrun, one process per GPU, NCCL): weak scaling on a box of N
stacked unit cubes along z (one cube's worth of DoFs per GPU), slab domain
decomposition with per-colour halo planes (paper_2405_19004_b200/dd.py).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")


def flops_per_patch(dim: int, k: int) -> int:
    """Algorithmic flops of the reference's per-patch contraction sequence
    (fastdiag.cpp:199-233 + :164-192 + smoother.cpp:119-120)."""
    ni, nc = 2 * k - 1, 2 * k + 1
    if dim == 3:
        return 4 * ni * nc ** 3 + 6 * ni ** 2 * nc ** 2 + 6 * ni ** 3 * nc + 12 * ni ** 4 + 3 * ni ** 3
    return 4 * ni * nc ** 2 + 4 * ni ** 2 * nc + 8 * ni ** 3 + 3 * ni ** 2


def algorithmic_bytes_per_step(dim: int, k: int, level: int, word: int) -> int:
    """x read once per colour + b^I read and x^I written once per patch
    (SURVEY.md §8d): w (2^d N + 2 P (2k-1)^d)."""
    n = 1 << level
    N = (n * k - 1) ** dim
    P = (n - 1) ** dim
    return word * ((1 << dim) * N + 2 * P * (2 * k - 1) ** dim)


def colour_patches(dim: int, level: int, color: int) -> int:
    n = 1 << level
    tot = 1
    for a in range(dim):
        tot *= n // 2 if (color >> a) & 1 else n // 2 - 1
    return tot


class ClockSampler:
    """NVML clocks / throttle reasons sampled in a thread (B200_PROFILING.md)."""

    REASONS = {
        "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4,
    }

    def __init__(self, device: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _sample(self):
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for name, bit in self.REASONS.items():
                if r & bit:
                    self.reasons.add(name)
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()
            self._sample()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_reference_run(args, steps: int, warmup: int, budget_s: float | None):
    """The reference's own CPU smooth (oracle/_ref = /root/reference compiled
    unmodified) with all host threads; returns (DoF/s, steps run, threads)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import refbind

    threads = os.cpu_count() or 1
    ref = refbind.RefMg(args.dim, args.degree, args.level, prec=0 if args.dtype == "f64" else 1,
                        variant=args.variant if args.variant in refbind.VARIANT else "fused", threads=threads)
    li = args.level - 1
    n = ref.n(li)
    x, b = refbind.fill_uniform(42, n, n)
    x = x.astype(ref.dtype)
    b = b.astype(ref.dtype)
    variant = args.variant if args.variant in refbind.VARIANT else "fused"
    vcode = refbind.VARIANT[variant]
    lib = refbind.lib()
    for _ in range(warmup):
        lib.ref_smooth(ref.h, li, vcode, refbind.P(x), refbind.P(b))
    done, t_total = 0, 0.0
    while True:
        t0 = time.perf_counter()
        st = lib.ref_smooth(ref.h, li, vcode, refbind.P(x), refbind.P(b))
        t_total += time.perf_counter() - t0
        assert st == 0
        done += 1
        if budget_s is None:
            if done >= steps:
                break
        elif t_total >= budget_s or done >= steps:
            break
    return n * done / t_total, done, threads, t_total


def run_reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    value, done, threads, t = cpu_reference_run(args, args.steps, args.warmup, None)
    out = {
        "impl": "reference",
        "metric": metric_name(args), "value": value, "unit": "DoF/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / done,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic", "config": config_dict(args),
        "cpu_baseline": {"value": value, "unit": "DoF/s", "cores": threads, "kind": "reference",
                         "sample": f"{done} full smoothing steps of the workload (pmg_ref::smooth<{args.dtype}>, "
                                   f"{args.variant}, threads={threads})"},
        "e2e": {"value": value, "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def smoother_kernel_name(args):
    """The kernel organisation pmg_smooth dispatches to (instantiate.cuh)."""
    if args.variant not in ("fused", "boundary"):
        return "vp_smooth_kernel"
    if args.degree == 1:
        return "vp_point_kernel"
    if args.dim == 3 and args.degree == 2:
        per_colour = ((1 << args.level) - 1) ** 3 / 8
        return "vp_patch3d_kernel" if per_colour >= 65536 else "vp_smooth_plane_kernel"
    if args.dim == 2 and (args.degree in (2, 3) or (args.degree == 4 and args.dtype == "f32")):
        return "vp_patch2d_kernel"
    if args.dim == 3 and (args.degree in (3, 4) or (args.degree in (5, 6) and args.dtype == "f32")):
        return "vp_smooth_pp_kernel"
    return "vp_smooth_kernel"


def metric_name(args):
    return f"DoF/s per smoother step ({args.variant} vertex-patch, {args.dtype})"


def config_dict(args):
    n = 1 << args.level
    return {"workload": f"{args.dim}D Q{args.degree} unit {'cube' if args.dim == 3 else 'square'}, "
                        f"2^{args.level} cells/dir, one {args.variant} smoother step",
            "dim": args.dim, "degree": args.degree, "level": args.level,
            "dofs": (n * args.degree - 1) ** args.dim, "patches": (n - 1) ** args.dim,
            "l2_flush": "256 MiB write before every timed step"}


# C3 (3D, ~1e8 DoF) and C4 (2D, ~2e8 DoF) finest levels per degree
C3_LEVELS = {1: 9, 2: 8, 3: 7, 4: 7, 5: 6, 6: 6, 7: 6}
C4_LEVELS = {1: 14, 2: 13, 3: 12, 4: 12, 5: 11, 6: 11, 7: 11}


def time_smoother(pmg, torch, lev, x, b, variant, steps, warmup, flush, stream):
    """Mean device time (s) of one smoothing step: W untimed steps, then K
    steps each bracketed by CUDA events with an L2 flush before each."""
    for _ in range(warmup):
        pmg.smooth(lev, x, b, variant)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.fill_(float(i))
        ev[i][0].record(stream)
        pmg.smooth(lev, x, b, variant)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(c) for a, c in ev) / 1e3 / steps


def sweep_entry(pmg, torch, dim, k, L, dtype, variant, steps, flush, stream, hbm_peak, max_mhz, sm_count,
                vcycle=False):
    """One configuration of a degree sweep: smoother step (and optionally one
    graph-captured V-cycle) with the same timing rules as the headline."""
    np_dt = np.float64 if dtype == "f64" else np.float32
    tdt = torch.float64 if dtype == "f64" else torch.float32
    word = 8 if dtype == "f64" else 4
    ctx = pmg.make_multigrid_context(dim, k, L, variant, dtype=np_dt)
    lev = ctx.levels[-1]
    N = lev.level.total_dofs
    gen = torch.Generator(device="cuda").manual_seed(7)
    x = torch.rand(N, dtype=tdt, device="cuda", generator=gen) * 2 - 1
    b = torch.rand(N, dtype=tdt, device="cuda", generator=gen) * 2 - 1
    t = time_smoother(pmg, torch, lev, x, b, variant, steps, 2, flush, stream)
    P = ((1 << L) - 1) ** dim
    flops = flops_per_patch(dim, k) * P
    byts = algorithmic_bytes_per_step(dim, k, L, word)
    fp_peak = sm_count * (64 if dtype == "f64" else 128) * 2 * max_mhz * 1e6
    e = {"dim": dim, "degree": k, "level": L, "dtype": dtype, "variant": variant, "dofs": N,
         "kernel": pmg.smoother_kernel(lev, variant, 0), "value": N / t, "unit": "DoF/s",
         "ms_per_step": t * 1e3, "fp_frac": flops / t / fp_peak, "hbm_frac": byts / t / (hbm_peak * 1e9)}
    if vcycle:
        li = L - 1
        pmg.v_cycle(ctx, li, x, b, use_graph=True)
        torch.cuda.synchronize()
        vt = 0.0
        for _ in range(3):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pmg.v_cycle(ctx, li, x, b, use_graph=True)
            e1.record(stream)
            torch.cuda.synchronize()
            vt += e0.elapsed_time(e1) / 1e3 / 3
        e["vcycle_value"] = N / vt
        e["vcycle_ms"] = vt * 1e3
    del x, b, ctx, lev
    torch.cuda.empty_cache()
    return e


def run_sweeps(args, pmg, torch, flush, stream, hbm_peak, max_mhz, sm_count):
    """C3 (3D Q1..Q7 ~1e8 DoF, f64 and f32, smoother step + V-cycle) and the
    "fused vs straightforward" comparison (BASELINE configs[3]: 2D Q1..Q7
    ~2e8 DoF; plus 3D Q2 / Q4): naive = the reference's per-patch body moved
    to the GPU directly (csrc/naive.cu, one CTA per patch, global-memory
    scratch); global = the reference's global variant on the device (level
    operator per colour into a global residual, then per-patch solves)."""
    K = args.sweep_steps
    common = (K, flush, stream, hbm_peak, max_mhz, sm_count)
    sweep = []
    for dtype in ("f64", "f32"):
        for k in range(1, 8):
            sweep.append(sweep_entry(pmg, torch, 3, k, C3_LEVELS[k], dtype, "fused", *common, vcycle=True))
    # C5 (3D Q4, 2^8 cells per direction, 1.07e9 DoF, 8.6 GB per f64 vector):
    # the multi-GPU configuration's whole problem on ONE B200 (the strong-
    # scaling baseline; weak-scaling unit = the Q4 L7 entry above)
    sweep.append(sweep_entry(pmg, torch, 3, 4, 8, "f64", "fused", *common, vcycle=True))
    comp = []
    cases = [(2, k, C4_LEVELS[k]) for k in range(1, 8)] + [(3, 2, 8), (3, 4, 7)]
    for dim, k, L in cases:
        fused = next((e for e in sweep if e["dim"] == dim and e["degree"] == k and e["level"] == L
                      and e["dtype"] == "f64"), None)
        if fused is None:
            fused = sweep_entry(pmg, torch, dim, k, L, "f64", "fused", *common)
        naive = sweep_entry(pmg, torch, dim, k, L, "f64", "naive", 2, *common[1:])
        # the reference's own straightforward variant (smoother.cpp:63-81): the
        # level operator over the whole level per colour, then the patch solves
        glob = sweep_entry(pmg, torch, dim, k, L, "f64", "global", 2, *common[1:])
        comp.append({"dim": dim, "degree": k, "level": L, "dofs": fused["dofs"], "dtype": "f64",
                     "fused": fused["value"], "fused_kernel": fused["kernel"], "naive": naive["value"],
                     "speedup": fused["value"] / naive["value"], "global": glob["value"],
                     "speedup_vs_global": fused["value"] / glob["value"], "unit": "DoF/s"})
    return comp, sweep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--degree", type=int, default=2)
    ap.add_argument("--level", type=int, default=6)
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--variant", default="fused")
    ap.add_argument("--cpu-budget", type=float, default=10.0, help="seconds of CPU reference work (cpu_baseline)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the C3/C4 degree sweeps and the naive comparator")
    ap.add_argument("--sweep-steps", type=int, default=5)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch

    import paper_2405_19004_b200 as pmg
    from paper_2405_19004_b200 import dd

    world, rank, local = dist_env()
    # PMG_DD_SHARED_GPU=1: all ranks on cuda:0 over gloo with host-staged halo
    # planes, to exercise the multi-rank path on a single-GPU box (test only)
    shared = os.environ.get("PMG_DD_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if args.dim != 3:
            raise SystemExit("multi-GPU slab decomposition is 3D only")

    dt = np.float64 if args.dtype == "f64" else np.float32
    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    word = 8 if args.dtype == "f64" else 4
    lib = pmg.load()
    ctx = pmg.make_multigrid_context(args.dim, args.degree, args.level, args.variant, dtype=dt, device=local)
    lev = ctx.levels[-1]
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    if world == 1:
        # the reference's unit cube on one GPU
        N_total = lev.level.total_dofs
        x = torch.rand(N_total, dtype=tdt, device="cuda", generator=gen) * 2 - 1
        b = torch.rand(N_total, dtype=tdt, device="cuda", generator=gen) * 2 - 1

        def step():
            pmg.smooth(lev, x, b, args.variant)

        colour_patch_counts = [colour_patches(args.dim, args.level, c) for c in range(1 << args.dim)]
    elif not shared:
        # weak scaling: a stack of `world` unit cubes along z, one slab per
        # GPU, driven by the library's C++ decomposition (pmg_dd_create_rank,
        # csrc/dd.cu): per colour the boundary-layer patches, one grouped
        # ncclSend/ncclRecv of k planes per interface on a side stream, the
        # interior patches concurrently
        nid = [pmg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        mctx = pmg.MultiGpuContext.for_rank(world, rank, local, nid[0], 3, args.degree, args.level, stack=world,
                                            dtype=dt, variant=args.variant)
        # the step (8 colours: boundary layers, grouped NCCL plane messages,
        # interiors) replayed as one captured CUDA graph
        if os.environ.get("PMG_DD_GRAPH", "1") == "1":
            mctx.set_graph(True)
        plan = dd.make_plan(world, rank, args.degree, args.level, stack=world)
        N_total = plan.m * plan.m * plan.mz
        x = mctx.slab_tensor(0, "x")
        b = mctx.slab_tensor(0, "b")
        x.copy_(torch.rand(x.numel(), dtype=tdt, device="cuda", generator=gen) * 2 - 1)
        b.copy_(torch.rand(b.numel(), dtype=tdt, device="cuda", generator=gen) * 2 - 1)
        torch.cuda.synchronize()
        stream = torch.cuda.ExternalStream(mctx.stream(0)[0])

        def step():
            mctx.smooth()

        graph_info = {"cuda_graph": os.environ.get("PMG_DD_GRAPH", "1") == "1"}
        l0 = lib.pmg_launch_count()
        step()  # the first call captures the graph: its launches are the step's
        mctx.synchronize()
        dd_step_launches = lib.pmg_launch_count() - l0

    else:
        # PMG_DD_SHARED_GPU: the Python driver (dd.py) over gloo, ranks sharing cuda:0
        plan = dd.make_plan(world, rank, args.degree, args.level, stack=world)
        N_total = plan.m * plan.m * plan.mz
        x = torch.rand(plan.nplanes * plan.plane_size, dtype=tdt, device="cuda", generator=gen) * 2 - 1
        b = torch.rand(plan.nplanes * plan.plane_size, dtype=tdt, device="cuda", generator=gen) * 2 - 1
        smoother = dd.SlabSmoother(plan, dd.gpu_kernel(lev, plan, x, b, args.variant),
                                   dd.StagedComm(x, plan.plane_size))

        def step():
            smoother.smooth()

    if world > 1:
        n = 1 << args.level
        colour_patch_counts = []
        for c in range(8):
            zb = (c >> 2) & 1
            nzv = sum(1 for v in range(plan.a, plan.b + 1) if v % 2 == zb)
            cnt = nzv
            for ax in range(2):
                cnt *= n // 2 if (c >> ax) & 1 else n // 2 - 1
            colour_patch_counts.append(cnt)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warm-up --------------------------------------------------------------
    for _ in range(args.warmup):
        step()
    barrier()

    timed_step, per_step_launches = step, None
    if world == 1 or shared:
        graph_info = None
    elif graph_info["cuda_graph"]:
        per_step_launches = dd_step_launches  # graph replays bypass the launch counter

    # ---- timed region: K steps, CUDA events per step, L2 flushed between ------
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = lib.pmg_launch_count()
    sampler = ClockSampler(local)
    with sampler, torch.cuda.stream(stream):  # N > 1: the decomposition's compute stream
        barrier()
        for i in range(args.steps):
            flush.fill_(float(i))
            ev[i][0].record(stream)
            timed_step()
            ev[i][1].record(stream)
        barrier()
    launches = lib.pmg_launch_count() - launches0
    if per_step_launches is not None:  # graph replays do not pass through the launch counter
        launches = per_step_launches * args.steps
    t_step = sum(a.elapsed_time(c) for a, c in ev) / 1e3 / args.steps
    if dist is not None:
        t = torch.tensor([t_step], dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_step = float(t.item())
    value = N_total / t_step

    # ---- roofline of the dominant kernel, from the TIMED steps -----------------
    # A step is exactly the 2^d colour launches of the smoother kernel and
    # nothing else (profiles/r02: ncu launch list of this command), so the
    # kernel's average launch duration is ms_per_step / launches per step and
    # its algorithmic bytes / flops per launch are the step's / launches per
    # step: achieved = algorithmic per step / t_step (no re-timed warm-L2 launches).
    F = flops_per_patch(args.dim, args.degree)
    step_flops = float(F * sum(colour_patch_counts))
    launches_per_step = sum(1 for c in colour_patch_counts if c)
    if world == 1:
        alg_bytes = algorithmic_bytes_per_step(args.dim, args.degree, args.level, word)
    else:  # this rank's slab: x read per colour + b^I read / x^I written per patch
        alg_bytes = word * ((1 << args.dim) * plan.nplanes * plan.plane_size
                            + 2 * sum(colour_patch_counts) * (2 * args.degree - 1) ** 3)
    peaks = json.load(open(MEASURED_PEAKS)) if os.path.exists(MEASURED_PEAKS) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    max_mhz = peaks.get("sm_max_mhz", 1965.0)
    fp_peak = sm_count * (64 if args.dtype == "f64" else 128) * 2 * max_mhz * 1e6 / 1e12
    traffic, traffic_note = None, None
    if world == 1 and os.path.exists(NCU_SUMMARY):  # the capture is of the single-GPU step
        try:
            s = json.load(open(NCU_SUMMARY))
            key = f"d{args.dim}k{args.degree}L{args.level}{args.dtype}{args.variant}"
            ent = s.get(key, {})
            if ent.get("dram_bytes_per_step"):
                traffic = float(ent["dram_bytes_per_step"]) / launches_per_step
                traffic_note = ent.get("note")
        except Exception:
            traffic = None
    kname = pmg.smoother_kernel(lev, args.variant, 0)
    roofline = {
        "bound": "hbm", "achieved": alg_bytes / t_step / 1e9, "peak": hbm_peak, "unit": "GB/s",
        "frac": alg_bytes / t_step / 1e9 / hbm_peak, "traffic": traffic,
        "traffic_note": traffic_note or "no ncu capture for this configuration",
        "kernel": kname + f" ({launches_per_step} launches per step = the whole step)",
        "algorithmic_bytes_per_launch": alg_bytes / launches_per_step,
        "launch_ms": t_step * 1e3 / launches_per_step,
        "algorithmic_bytes_per_step": alg_bytes,
        "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if "hbm_gbs" in peaks else "fallback 6650 GB/s",
    }
    roofline_fp = {
        "bound": f"{args.dtype} CUDA-core FMA", "achieved": step_flops / t_step / 1e12,
        "peak": fp_peak, "unit": "TFLOP/s", "frac": step_flops / t_step / 1e12 / fp_peak,
        "algorithmic_flops_per_patch": F, "algorithmic_flops_per_launch": step_flops / launches_per_step,
        "peak_source": f"{sm_count} SMs x {64 if args.dtype == 'f64' else 128} FMA/clk x 2 x {max_mhz} MHz",
    }
    # which roofline binds: at sizes whose x and b fit in L2 (C2: 2 x 16 MiB of
    # 126 MB) only the first colour of a step reads HBM, so the FP pipe (and
    # the issue rate) is the limit, not HBM
    fits_l2 = 2 * N_total * word < 100e6
    ridge = fp_peak * 1e12 / (hbm_peak * 1e9)  # flop/B
    binding = "roofline" if (not fits_l2 and step_flops / alg_bytes < ridge) else "roofline_fp"

    # ---- V-cycle throughput (secondary metric, single GPU) ---------------------
    vcycle = None
    if world == 1:
        li = args.level - 1
        pmg.v_cycle(ctx, li, x, b, use_graph=True)
        torch.cuda.synchronize()
        vreps = max(3, min(10, args.steps))
        vt = 0.0
        for _ in range(vreps):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pmg.v_cycle(ctx, li, x, b, use_graph=True)
            e1.record(stream)
            torch.cuda.synchronize()
            vt += e0.elapsed_time(e1) / 1e3
        vt /= vreps
        vcycle = {"value": N_total / vt, "unit": "DoF/s", "ms": vt * 1e3, "cuda_graph": True}
    elif not shared:
        # the decomposed V-cycle of the reference's unit cube at the same level
        # (strong scaling of the secondary metric; one graph per rank)
        nid = [pmg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        vctx = pmg.MultiGpuContext.for_rank(world, rank, local, nid[0], 3, args.degree, args.level, stack=1,
                                            dtype=dt, variant=args.variant)
        vctx.set_graph(True)
        vx, vb = vctx.slab_tensor(0, "x"), vctx.slab_tensor(0, "b")
        vx.copy_(torch.rand(vx.numel(), dtype=tdt, device="cuda", generator=gen) * 2 - 1)
        vb.copy_(torch.rand(vb.numel(), dtype=tdt, device="cuda", generator=gen) * 2 - 1)
        vstream = torch.cuda.ExternalStream(vctx.stream(0)[0])
        vctx.v_cycle()
        vctx.synchronize()
        vreps = max(3, min(10, args.steps))
        vt = 0.0
        with torch.cuda.stream(vstream):
            for _ in range(vreps):
                barrier()
                flush.fill_(1.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(vstream)
                vctx.v_cycle()
                e1.record(vstream)
                torch.cuda.synchronize()
                vt += e0.elapsed_time(e1) / 1e3
        t = torch.tensor([vt / vreps], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        vt = float(t.item())
        nv = ((1 << args.level) * args.degree - 1) ** 3
        vcycle = {"value": nv / vt, "unit": "DoF/s", "ms": vt * 1e3, "cuda_graph": True, "scaling": "strong",
                  "workload": f"unit cube 2^{args.level} cells/dir over {world} z-slabs (pmg_dd_v_cycle)"}
        del vctx

    # ---- e2e through the public API with host buffers (pinned) -----------------
    e2e_steps = max(3, min(args.steps, 20))
    if world == 1:
        xh = torch.empty(N_total, dtype=tdt, pin_memory=True).numpy()
        bh = torch.empty(N_total, dtype=tdt, pin_memory=True).numpy()
        xh[:] = x.cpu().numpy()
        bh[:] = b.cpu().numpy()
        # the reference-facing C-ABI call itself (what the reference's smooth<T>
        # forwards to): pmg_smooth_host(level, variant, x, b)
        # = H2D of x, b, the colour kernels, D2H of x (pipelined)
        import ctypes

        from paper_2405_19004_b200._lib import VARIANTS

        hx, hb, vcode = ctypes.c_void_p(xh.ctypes.data), ctypes.c_void_p(bh.ctypes.data), VARIANTS[args.variant]
        for _ in range(2):
            assert lib.pmg_smooth_host(lev.handle, vcode, hx, hb) == 0, lib.pmg_last_error()
        barrier()
        st = 0
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            st |= lib.pmg_smooth_host(lev.handle, vcode, hx, hb)
        t_e2e = (time.perf_counter() - t0) / e2e_steps
        assert st == 0, lib.pmg_last_error()
        h2d, d2h = 2 * N_total * word, N_total * word
    else:
        xh = torch.empty(x.numel(), dtype=tdt, pin_memory=True)
        bh = torch.empty(b.numel(), dtype=tdt, pin_memory=True)
        xh.copy_(x)
        bh.copy_(b)
        own = dd.owned_part(plan, x)
        oh = torch.empty(own.numel(), dtype=tdt, pin_memory=True)
        barrier()
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            for _ in range(e2e_steps):
                x.copy_(xh, non_blocking=True)
                b.copy_(bh, non_blocking=True)
                step()
                oh.copy_(dd.owned_part(plan, x), non_blocking=True)
                torch.cuda.synchronize()
        t_e2e = (time.perf_counter() - t0) / e2e_steps
        h2d, d2h = (xh.numel() + bh.numel()) * word, oh.numel() * word
    if dist is not None:
        t = torch.tensor([t_e2e], dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_e2e = float(t.item())

    cfg = config_dict(args)
    if world > 1:
        cfg["workload"] = (f"3D Q{args.degree} box of {world} stacked unit cubes (2^{args.level} cells/dir each), "
                           f"one {args.variant} smoother step, z-slab per GPU")
        cfg["dofs"] = N_total
        cfg["parallelism"] = (f"slab decomposition x{world} (C++ pmg_dd_*, NCCL halo planes per colour)" if not shared
                              else f"slab decomposition x{world} (dd.py over gloo, ranks sharing one GPU)")
        if graph_info is not None:
            cfg["dd_step"] = graph_info
    out = {
        "metric": metric_name(args), "value": value, "unit": "DoF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (x, b ~ U(-1,1))", "config": cfg,
        "roofline": roofline, "roofline_fp": roofline_fp, "roofline_binding": binding,
        "e2e": {"value": N_total / t_e2e, "unit": "DoF/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "api": "pmg_smooth_host (C-ABI, pinned host buffers)" if world == 1 else
                       "slab H2D, pmg_dd_smooth (C-ABI), owned-plane D2H (pinned)"},
        "clocks": sampler.summary(), "gpu_launches": int(launches),
    }
    if vcycle is not None:
        out["vcycle"] = vcycle
    if world == 1 and not args.no_sweep:
        del x, b, xh, bh
        ctx = lev = None
        torch.cuda.empty_cache()
        out["comparator"], out["sweep"] = run_sweeps(args, pmg, torch, flush, stream, hbm_peak, max_mhz, sm_count)

    if rank == 0 and world == 1 and not args.no_cpu:
        v, done, threads, tcpu = cpu_reference_run(args, 10 ** 6, 1, args.cpu_budget)
        out["cpu_baseline"] = {"value": v, "unit": "DoF/s", "cores": threads, "kind": "reference",
                               "sample": f"{done} full smoothing steps of the same workload in {tcpu:.1f} s "
                                         f"(oracle/_ref = /root/reference compiled unmodified, threads={threads})"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
