"""Paper table "vertex patch vs point Gauss-Seidel": 3D
Q1..Q7, f = 1, V-cycles (1 pre / 1 post smoothing) with the vertex-patch
smoother or one lexicographic point Gauss-Seidel sweep (kind point_gs, the
device wavefront sweep) per smoothing step. Reported: plain V-cycle
iterations from x = 0 to ||r|| <= 1e-9 ||b|| (the paper's count), and the
reference's full_multigrid while-loop count at the same tolerance. Levels:
the two finest the reference's 1e7-nonzero CSR budget admits for point GS.

python tools/gs_table.py > profiles/r02/gs_table.txt"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2405_19004_b200 as pmg  # noqa: E402


def vcycle_iterations(mg, b, tol=1e-9, cap=200):
    lev = mg.levels[-1]
    x = torch.zeros_like(b)
    r = torch.empty_like(b)
    b0 = pmg.vector_norm(b)
    its = 0
    while True:
        pmg.compute_residual(lev, x, b, r)
        if pmg.vector_norm(r) <= tol * b0 or its >= cap:
            return its
        pmg.v_cycle(mg, len(mg.levels) - 1, x, b)
        its += 1


print("3D Poisson, f = 1, tolerance 1e-9 relative to ||b||")
print(f"{'k':>2} {'L':>2} {'DoF':>9} | {'V-cycles: patch':>16} {'point GS':>9} | {'FMG: patch':>11} {'point GS':>9}"
      f" | {'GS V-cycle ms':>13}")
for k in range(1, 8):
    levels = []
    for L in range(8, 0, -1):
        try:
            pmg.make_multigrid_context(3, k, L, kind="point_gs")
        except RuntimeError:
            continue
        levels.append(L)
        if len(levels) == 2:
            break
    for L in sorted(levels):
        hier = pmg.build_hierarchy(3, k, L)
        rhs = [pmg.compute_rhs(lev, "one") for lev in hier]
        bd = torch.from_numpy(rhs[-1]).cuda()
        vc, fm, ms = [], [], 0.0
        for kind in ("vertex_patch", "point_gs"):
            mg = pmg.make_multigrid_context(3, k, L, kind=kind)
            vc.append(vcycle_iterations(mg, bd))
            x = np.zeros(hier[-1].total_dofs)
            fm.append(pmg.full_multigrid(mg, rhs, x, 1e-9, max_iterations=200).iterations)
            if kind == "point_gs":
                xd = torch.zeros_like(bd)
                pmg.v_cycle(mg, L - 1, xd, bd)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for _ in range(5):
                    pmg.v_cycle(mg, L - 1, xd, bd)
                torch.cuda.synchronize()
                ms = (time.perf_counter() - t0) / 5 * 1e3
        print(f"{k:>2} {L:>2} {hier[-1].total_dofs:>9} | {vc[0]:>16} {vc[1]:>9} | {fm[0]:>11} {fm[1]:>9} | {ms:>13.2f}")
print("paper (3D V-cycles, levels where the counts are constant): point GS 6 8 11 13 19 20 27 30, "
      "vertex patch 6 5 3 3 3 3 2 2 (Q1..Q8)")
