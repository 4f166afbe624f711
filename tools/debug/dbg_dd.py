import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2405_19004_b200 as pmg
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for L in (4, 5):
    mg = pmg.make_multigrid_context(3, k, L)
    n = mg.levels[-1].level.total_dofs
    rng = np.random.default_rng(1)
    data = {"random": (rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)),
            "smooth": (np.zeros(n), pmg.compute_rhs(mg.levels[-1].level, "one"))}
    for P in (1, 2, 3):
        try:
            ctx = pmg.MultiGpuContext([0] * P, 3, k, L)
        except ValueError as e:
            print(L, P, "skip", e); continue
        for name, (x0, b) in data.items():
            xs = torch.from_numpy(x0.copy()).cuda(); bd = torch.from_numpy(b).cuda()
            pmg.smooth(mg.levels[-1], xs, bd, "fused")
            ctx.scatter("x", x0.copy()); ctx.scatter("b", b.copy()); ctx.smooth()
            d_s = np.abs(ctx.gather("x") - xs.cpu().numpy()).max()
            xv = torch.from_numpy(x0.copy()).cuda(); pmg.v_cycle(mg, L - 1, xv, bd)
            ctx.scatter("x", x0.copy()); ctx.v_cycle()
            d_v = np.abs(ctx.gather("x") - xv.cpu().numpy()).max()
            print(f"k={k} L={L} P={P} dd_levels={ctx.decomposed_levels} {name}: smooth {d_s:.2e} vcycle {d_v:.2e}")
