import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2405_19004_b200 as pmg
from paper_2405_19004_b200._lib import DivergenceError
k, L, P = 2, 4, 1
rhs = [pmg.compute_rhs(lev, "one") for lev in pmg.build_hierarchy(3, k, L)]
mg = pmg.make_multigrid_context(3, k, L)
R = [torch.from_numpy(r).cuda() for r in rhs]
def z(li): return torch.zeros(rhs[li].size, dtype=torch.float64, device="cuda")
def nested(skip_last=False, vc_counts=None):
    x = z(0); pmg.v_cycle(mg, 0, x, R[0])
    for li in range(1, L):
        xn = z(li); pmg.prolongate(mg.levels[li-1], mg.levels[li], x, xn)
        n = 1 if vc_counts is None else vc_counts[li]
        for _ in range(n):
            pmg.v_cycle(mg, li, xn, R[li])
        x = xn
    return x.cpu().numpy()
ctx = pmg.MultiGpuContext([0] * P, 3, k, L)
try:
    ctx.full_multigrid(rhs, 1e-8, max_iterations=0)
except DivergenceError:
    pass
xdd = ctx.gather("x")
cands = {"single": nested(), "last0": nested(vc_counts=[1,1,1,0]), "last2": nested(vc_counts=[1,1,1,2]),
         "l3_0": nested(vc_counts=[1,1,0,1]), "l3_2": nested(vc_counts=[1,1,2,1]), "l2_0": nested(vc_counts=[1,0,1,1])}
for n, c in cands.items():
    print(n, np.abs(c - xdd).max())
# V-cycle of the dd context on the single's P x3 vs the single's V-cycle
x = z(0); pmg.v_cycle(mg, 0, x, R[0])
for li in range(1, L - 1):
    xn = z(li); pmg.prolongate(mg.levels[li-1], mg.levels[li], x, xn); pmg.v_cycle(mg, li, xn, R[li]); x = xn
xp = z(L - 1); pmg.prolongate(mg.levels[L-2], mg.levels[L-1], x, xp)
xpn = xp.cpu().numpy()
ctx.scatter("x", xpn.copy()); ctx.scatter("b", rhs[-1])
ctx.v_cycle()
xs = xp.clone(); pmg.v_cycle(mg, L - 1, xs, R[L-1])
print("dd vcycle on P x3 vs single:", np.abs(ctx.gather("x") - xs.cpu().numpy()).max())
ctx2 = pmg.MultiGpuContext([0] * P, 3, k, L)
try:
    ctx2.full_multigrid(rhs, 1e-8, max_iterations=0)
except DivergenceError:
    pass
print("fresh ctx fmg vs first:", np.abs(ctx2.gather("x") - xdd).max())
ctx2.scatter("x", xpn.copy()); ctx2.scatter("b", rhs[-1]); ctx2.v_cycle()
print("after fmg, dd vcycle on P x3 vs single:", np.abs(ctx2.gather("x") - xs.cpu().numpy()).max())
