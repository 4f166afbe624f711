"""One eager V-cycle inside an NVTX range "vc" (for an ncu launch list of
the V-cycle's kernels: ncu --nvtx --nvtx-include "vc/" ...).

python tools/debug/vc_kernels.py dim k L dtype
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2405_19004_b200 as pmg  # noqa: E402

dim, k, L, dtype = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
if os.environ.get("PMG_IMPL"):
    pmg.set_smoother_impl(os.environ["PMG_IMPL"])
dt = np.float64 if dtype == "f64" else np.float32
tdt = torch.float64 if dtype == "f64" else torch.float32
ctx = pmg.make_multigrid_context(dim, k, L, "fused", dtype=dt)
n = ctx.levels[-1].level.total_dofs
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand(n, dtype=tdt, device="cuda", generator=g)
b = torch.rand(n, dtype=tdt, device="cuda", generator=g)
for _ in range(2):
    pmg.v_cycle(ctx, L - 1, x, b)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("vc")
pmg.v_cycle(ctx, L - 1, x, b)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
