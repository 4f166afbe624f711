"""Generate the golden fixtures from the REFERENCE itself (test infrastructure).

Runs the unmodified reference library compiled from /root/reference into
oracle/_ref/libpmg_ref.so (oracle/Makefile) and stores its outputs for small
seeded problems in tests/golden/*.npz:

  inputs  x0, b   std::mt19937_64(42), U(-1,1), x0 filled first then b
  smooth_<variant>  pmg_ref::smooth<T>(ctx, x0, b, variant)
  residual          pmg_ref::compute_residual<T>(ctx, x0, b)
  laplacian         pmg_ref::apply_laplacian<T>(x0)
  vcycle            pmg_ref::v_cycle<T>(ctx, L-1, x0, b)
  prolongate / restrict on level L-1 -> L from seeded coarse / fine vectors
  fmg_<rhs>         pmg_ref::full_multigrid (f64): iterations + history, with
                    the reference's own compute_rhs per level

Usage: python tests/golden/make_golden.py   (needs oracle/_ref built here)
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import refbind  # noqa: E402

CASES = [
    # (name, dim, k, L, prec)
    ("c1_2d_q2_l6_f64", 2, 2, 6, 0),
    ("2d_q1_l4_f64", 2, 1, 4, 0),
    ("2d_q7_l3_f64", 2, 7, 3, 0),
    ("3d_q1_l4_f64", 3, 1, 4, 0),
    ("3d_q2_l3_f64", 3, 2, 3, 0),
    ("3d_q4_l2_f64", 3, 4, 2, 0),
    ("3d_q7_l2_f64", 3, 7, 2, 0),
    ("3d_q3_l3_f32", 3, 3, 3, 1),
    ("2d_q4_l4_f32", 2, 4, 4, 1),
]


def main():
    assert refbind.available(), "oracle/_ref/libpmg_ref.so missing: make -C oracle"
    for name, dim, k, L, prec in CASES:
        ref = refbind.RefMg(dim, k, L, prec=prec)
        dt = ref.dtype
        n = ref.n(L - 1)
        x0, b = refbind.fill_uniform(42, n, n)
        x0, b = x0.astype(dt), b.astype(dt)
        out = {"dim": dim, "k": k, "L": L, "prec": prec, "x0": x0, "b": b}
        for v in refbind.VARIANT:
            out[f"smooth_{v}"] = ref.smooth(L - 1, x0, b, v)
        out["residual"] = ref.residual(L - 1, x0, b)
        out["laplacian"] = ref.apply_laplacian(L - 1, x0)
        out["vcycle"] = ref.vcycle(L - 1, x0, b)
        if L >= 2:
            nc = ref.n(L - 2)
            xc, rf = refbind.fill_uniform(7, nc, n)
            xc, rf = xc.astype(dt), rf.astype(dt)
            out["xc"], out["rf"] = xc, rf
            out["prolongate"] = ref.prolongate(L - 2, xc)
            out["restrict"] = ref.restrict(L - 2, rf)
        if prec == 0 and n <= 20000:
            for kind, tag in ((0, "one"), (1, "sin")):
                st, x, it, hist = ref.fmg(kind, 1e-8)
                assert st == 0
                out[f"fmg_{tag}_iterations"] = it
                out[f"fmg_{tag}_history"] = hist
                out[f"fmg_{tag}_x"] = x
                out[f"rhs_{tag}"] = refbind.compute_rhs(dim, k, L, kind)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print(name, n, "ok")


if __name__ == "__main__":
    main()
