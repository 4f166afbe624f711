"""V-cycle time per finest level (development helper): the increments
T(L) - T(L-1) show what each level adds, i.e. where the coarse levels are
latency- rather than bandwidth-bound.

python tools/vcycle_levels.py dim k Lmax dtype [reps]
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_19004_b200 as pmg  # noqa: E402


def vtime(dim, k, L, dtype, reps):
    dt = np.float64 if dtype == "f64" else np.float32
    tdt = torch.float64 if dtype == "f64" else torch.float32
    ctx = pmg.make_multigrid_context(dim, k, L, "fused", dtype=dt)
    n = ctx.levels[-1].level.total_dofs
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand(n, dtype=tdt, device="cuda", generator=g)
    b = torch.rand(n, dtype=tdt, device="cuda", generator=g)
    for _ in range(3):
        pmg.v_cycle(ctx, L - 1, x, b, use_graph=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        pmg.v_cycle(ctx, L - 1, x, b, use_graph=True)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps
    del ctx
    return n, t


if __name__ == "__main__":
    dim, k, Lmax, dtype = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 50
    prev = 0.0
    tag = os.environ.get("PMG_SWEEP_AUTO_TILES", "0")
    for L in range(1, Lmax + 1):
        n, t = vtime(dim, k, L, dtype, reps)
        print(f"[sweep_tiles={tag}] d={dim} k={k} L={L} {dtype} N={n:10d} vcycle {t*1e3:8.1f} us  "
              f"(+{(t - prev)*1e3:7.1f} us)  {n / t / 1e6:7.3f} GDoF/s", flush=True)
        prev = t
