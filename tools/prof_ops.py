"""Minimal workload for ncu: residual / restrict / prolong of one config.
python tools/prof_ops.py dim k L dtype"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_19004_b200 as pmg  # noqa: E402
dim, k, L, dtype = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
dt = np.float64 if dtype == "f64" else np.float32
tdt = torch.float64 if dtype == "f64" else torch.float32
ctx = pmg.make_multigrid_context(dim, k, L, "fused", dtype=dt)
f, c = ctx.levels[-1], ctx.levels[-2]
x = torch.rand(f.level.total_dofs, dtype=tdt, device="cuda"); b = torch.rand_like(x); r = torch.empty_like(x)
xc = torch.rand(c.level.total_dofs, dtype=tdt, device="cuda")
for _ in range(2):
    pmg.compute_residual(f, x, b, r); pmg.restrict_vector(c, f, x, xc); pmg.prolongate(c, f, xc, x, accumulate=True)
torch.cuda.synchronize()
