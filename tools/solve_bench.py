"""Mixed vs double precision GMRES + V-cycle solves of the 3D Poisson problem
with u = prod sin(pi x_a) (the paper's Table: GMRES in f64
right-preconditioned by one V-cycle with one pre- and post-smoothing step in
f32 or f64, relative residual reduction 1e-9), on one B200.

python tools/solve_bench.py [k L restart ...]     (default: 7 7 4  3 8 6  1 9 10)
Prints one JSON line per (degree, mode); time = device-synchronised GMRES
wall time (setup and right-hand side assembly excluded, as in the paper).
"""

import gc
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_19004_b200 as pmg  # noqa: E402

PAPER = {1: (135e6, 1.12e-06, 5, 3.391, 2.385), 3: (454e6, 2.30e-13, 3, 3.941, 2.418),
         7: (721e6, 2.89e-16, 2, 5.891, 3.326)}


def run(k, L, restart, tol=1e-9):
    op = pmg.make_multigrid_context(3, k, L, "fused", dtype=np.float64)
    lev = op.levels[-1]
    n = lev.level.total_dofs
    b = torch.empty(n, dtype=torch.float64, device="cuda")
    pmg.compute_rhs_device(lev, "sin", b)
    out = []
    for mode in ["double", "mixed"]:
        prec = op if mode == "double" else pmg.make_multigrid_context(3, k, L, "fused", dtype=np.float32)
        x = torch.zeros(n, dtype=torch.float64, device="cuda")
        pmg.gmres(op, prec, b, x, tol, restart=restart, max_iterations=50)  # warm-up (graphs, workspaces)
        x.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = pmg.gmres(op, prec, b, x, tol, restart=restart, max_iterations=50)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        err = pmg.l2_error(lev, x)
        rec = {"degree": k, "level": L, "dofs": n, "mode": mode, "iterations": st.iterations,
               "time_s": t, "l2_error": err, "restart": restart, "tol": tol,
               "residual_history": st.residual_history}
        if k in PAPER:
            p = PAPER[k]
            rec["paper_a100"] = {"dofs": p[0], "l2_error": p[1], "iterations": p[2],
                                 "time_s": p[3] if mode == "double" else p[4]}
        out.append(rec)
        print(json.dumps(rec), flush=True)
        del prec, x
        gc.collect()
        torch.cuda.empty_cache()
    print(json.dumps({"degree": k, "speedup_mixed_over_double": out[0]["time_s"] / out[1]["time_s"]}), flush=True)


if __name__ == "__main__":
    a = [int(v) for v in sys.argv[1:]] or [7, 7, 4, 3, 8, 6, 1, 9, 10]
    for i in range(0, len(a), 3):
        run(a[i], a[i + 1], a[i + 2])
        gc.collect()  # contexts hold their levels (and the GMRES workspace) in a cycle
        torch.cuda.empty_cache()
