"""Device timing of the V-cycle's non-smoother kernels against their HBM roofline
(development helper): residual r = b - A x, restriction, prolongation (+=).

python tools/quick_ops.py dim k L dtype [dim k L dtype ...]
"""

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_19004_b200 as pmg  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6556.0) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6556.0


def timeit(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def run(dim, k, L, dtype):
    dt = np.float64 if dtype == "f64" else np.float32
    tdt = torch.float64 if dtype == "f64" else torch.float32
    w = 8 if dtype == "f64" else 4
    ctx = pmg.make_multigrid_context(dim, k, L, "fused", dtype=dt)
    f, c = ctx.levels[-1], ctx.levels[-2]
    nf, nc = f.level.total_dofs, c.level.total_dofs
    x = torch.rand(nf, dtype=tdt, device="cuda")
    b = torch.rand(nf, dtype=tdt, device="cuda")
    r = torch.empty_like(x)
    xc = torch.rand(nc, dtype=tdt, device="cuda")
    t = timeit(lambda: pmg.compute_residual(f, x, b, r))
    print(f"d={dim} k={k} L={L} {dtype} N={nf:.3e}  residual {t*1e3:7.3f} ms {3*nf*w/t/1e9:7.0f} GB/s "
          f"({100*3*nf*w/t/1e9/PEAK:4.1f}% HBM)", end="")
    t = timeit(lambda: pmg.restrict_vector(c, f, x, xc))
    print(f" | restrict {t*1e3:7.3f} ms {(nf+nc)*w/t/1e9:7.0f} GB/s ({100*(nf+nc)*w/t/1e9/PEAK:4.1f}%)", end="")
    t = timeit(lambda: pmg.prolongate(c, f, xc, x, accumulate=True))
    print(f" | prolong+= {t*1e3:7.3f} ms {(2*nf+nc)*w/t/1e9:7.0f} GB/s ({100*(2*nf+nc)*w/t/1e9/PEAK:4.1f}%)",
          flush=True)


if __name__ == "__main__":
    a = sys.argv[1:]
    cfgs = [(int(a[i]), int(a[i + 1]), int(a[i + 2]), a[i + 3]) for i in range(0, len(a), 4)]
    for cfg in cfgs:
        run(*cfg)
