"""Minimal workload for ncu: a few smoothing steps / V-cycles of one config.

python tools/prof_target.py dim k L dtype variant [n_smooth] [n_vcycle]
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_19004_b200 as pmg  # noqa: E402

dim, k, L = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dtype = sys.argv[4] if len(sys.argv) > 4 else "f64"
variant = sys.argv[5] if len(sys.argv) > 5 else "fused"
ns = int(sys.argv[6]) if len(sys.argv) > 6 else 3
if os.environ.get("PMG_IMPL"):
    pmg.set_smoother_impl(os.environ["PMG_IMPL"])
nv = int(sys.argv[7]) if len(sys.argv) > 7 else 0
dt = np.float64 if dtype == "f64" else np.float32
tdt = torch.float64 if dtype == "f64" else torch.float32
ctx = pmg.make_multigrid_context(dim, k, L, variant, dtype=dt)
lev = ctx.levels[-1]
n = lev.level.total_dofs
x = torch.rand(n, dtype=tdt, device="cuda") * 2 - 1
b = torch.rand(n, dtype=tdt, device="cuda") * 2 - 1
for _ in range(ns):
    pmg.smooth(lev, x, b, variant)
for _ in range(nv):
    pmg.v_cycle(ctx, L - 1, x, b)
torch.cuda.synchronize()
print("done", n)
