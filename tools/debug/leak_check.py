"""Create / use / destroy multigrid contexts repeatedly and watch free device memory."""
import gc
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2405_19004_b200 as pmg  # noqa: E402

torch.cuda.init()
free0 = torch.cuda.mem_get_info()[0]
for it in range(12):
    for (k, L, dt) in [(2, 5, np.float64), (1, 5, np.float32), (4, 3, np.float64)]:
        ctx = pmg.make_multigrid_context(3, k, L, dtype=dt)
        n = ctx.levels[-1].level.total_dofs
        x = torch.zeros(n, dtype=torch.float64 if dt == np.float64 else torch.float32, device="cuda")
        b = torch.ones_like(x)
        pmg.smooth(ctx.levels[-1], x, b, "fused")
        pmg.v_cycle(ctx, L - 1, x, b, use_graph=True)
        pmg.v_cycle(ctx, L - 1, x, b, use_graph=False)
        if dt == np.float64:
            pmg.smooth_host(ctx.levels[-1], x.cpu().numpy(), b.cpu().numpy(), "fused") if hasattr(pmg, "smooth_host") else None
        del ctx, x, b
        gc.collect()
    torch.cuda.synchronize()
    free = torch.cuda.mem_get_info()[0]
    print(f"iter {it}: free {free / 2**20:.0f} MiB (delta {(free0 - free) / 2**20:+.0f} MiB)", flush=True)
