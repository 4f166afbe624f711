"""Time the C++ slab decomposition (pmg_dd_*) with P virtual ranks sharing one
GPU against the single-device smoother / V-cycle (same level): the cost of the
decomposition's extra launches, events and plane copies when there is no
second GPU to absorb the work. Host wall clock around a synchronised loop.

python tools/dd_time.py [k L]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2405_19004_b200 as pmg  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
L = int(sys.argv[2]) if len(sys.argv) > 2 else 7
reps = 20
mg = pmg.make_multigrid_context(3, k, L)
n = mg.levels[-1].level.total_dofs
x = torch.rand(n, dtype=torch.float64, device="cuda")
b = torch.rand(n, dtype=torch.float64, device="cuda")


def tm(f, sync):
    for _ in range(3):
        f()
    sync()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    sync()
    return (time.perf_counter() - t0) / reps * 1e3


ts = tm(lambda: pmg.smooth(mg.levels[-1], x, b), torch.cuda.synchronize)
tv = tm(lambda: pmg.v_cycle(mg, L - 1, x, b, use_graph=True), torch.cuda.synchronize)
print(f"3D Q{k} L{L} ({n:.3e} DoF) single device: smooth {ts:.3f} ms, V-cycle (graph) {tv:.3f} ms")
xh, bh = x.cpu().numpy(), b.cpu().numpy()
for P in (1, 2, 4, 8):
    try:
        ctx = pmg.MultiGpuContext([0] * P, 3, k, L)
    except ValueError as e:
        print(f"P={P}: {e}")
        continue
    ctx.scatter("x", xh)
    ctx.scatter("b", bh)
    s = tm(ctx.smooth, ctx.synchronize)
    v = tm(ctx.v_cycle, ctx.synchronize)
    ctx.set_graph(True)
    sg = tm(ctx.smooth, ctx.synchronize)
    vg = tm(ctx.v_cycle, ctx.synchronize)
    print(f"P={P} virtual ranks (decomposed levels {ctx.decomposed_levels}): smooth {s:.3f} ms "
          f"({ts / s:.2f}x single), as one graph {sg:.3f} ms ({ts / sg:.2f}x); V-cycle {v:.3f} ms "
          f"({tv / v:.2f}x single), as one graph {vg:.3f} ms ({tv / vg:.2f}x)")
    del ctx
