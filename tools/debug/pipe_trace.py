import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2405_19004_b200 as pmg
lev = pmg.make_level_context(pmg.build_hierarchy(3, 2, 6)[-1])
n = lev.level.total_dofs
xh = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy(); xh[:] = 0.5
bh = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy(); bh[:] = 0.25
for i in range(4):
    print("call", i, file=sys.stderr)
    pmg.smooth(lev, xh, bh, "fused")
