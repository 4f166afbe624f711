"""Quick device timing of the smoother / V-cycle (development helper).

python tools/quick_time.py [dim k L dtype variant] ...
"""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_19004_b200 as pmg  # noqa: E402


def flops_per_patch(dim, k):
    ni, nc = 2 * k - 1, 2 * k + 1
    if dim == 3:
        return 4 * ni * nc ** 3 + 6 * ni ** 2 * nc ** 2 + 6 * ni ** 3 * nc + 12 * ni ** 4 + 3 * ni ** 3
    return 4 * ni * nc ** 2 + 4 * ni ** 2 * nc + 8 * ni ** 3 + 3 * ni ** 2


def run(dim, k, L, dtype, variant, reps=10):
    dt = np.float64 if dtype == "f64" else np.float32
    tdt = torch.float64 if dtype == "f64" else torch.float32
    ctx = pmg.make_multigrid_context(dim, k, L, variant, dtype=dt)
    lev = ctx.levels[-1]
    n = lev.level.total_dofs
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand(n, dtype=tdt, device="cuda", generator=g) * 2 - 1
    b = torch.rand(n, dtype=tdt, device="cuda", generator=g) * 2 - 1
    for _ in range(3):
        pmg.smooth(lev, x, b, variant)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        pmg.smooth(lev, x, b, variant)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    patches = ((1 << L) - 1) ** dim
    fl = flops_per_patch(dim, k) * patches / t
    peak = (148 * (64 if dtype == "f64" else 128) * 2 * 1.965e9)
    # v-cycle
    for _ in range(2):
        pmg.v_cycle(ctx, L - 1, x, b, use_graph=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        pmg.v_cycle(ctx, L - 1, x, b, use_graph=True)
    e1.record()
    torch.cuda.synchronize()
    tv = e0.elapsed_time(e1) / reps / 1e3
    print(f"d={dim} k={k} L={L} {dtype} {variant:9s} N={n:.3e}  smooth {t*1e3:8.3f} ms  {n/t/1e9:7.3f} GDoF/s  "
          f"{fl/1e12:6.2f} TF ({100*fl/peak:5.1f}% of {peak/1e12:.1f})  vcycle {tv*1e3:8.3f} ms {n/tv/1e9:7.3f} GDoF/s",
          flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    if not args:
        cfgs = [(3, 2, 6, "f64", "fused"), (3, 2, 6, "f64", "naive"), (3, 2, 6, "f64", "global"),
                (3, 4, 7, "f64", "fused"), (3, 4, 7, "f32", "fused"), (3, 4, 6, "f64", "naive"),
                (3, 1, 8, "f64", "fused"), (3, 3, 7, "f64", "fused"), (3, 5, 6, "f64", "fused"),
                (3, 6, 6, "f64", "fused"), (3, 7, 6, "f64", "fused"), (2, 7, 10, "f64", "fused"),
                (2, 4, 11, "f64", "fused")]
    else:
        cfgs = [(int(args[i]), int(args[i + 1]), int(args[i + 2]), args[i + 3], args[i + 4])
                for i in range(0, len(args), 5)]
    impls = os.environ.get("PMG_IMPLS", "auto").split(",")
    for c in cfgs:
        for impl in impls:
            pmg.set_smoother_impl(impl)
            print(f"[{impl}] ", end="")
            run(*c)
