"""ctypes binding of the reference library built into oracle/_ref (TEST INFRA).

oracle/_ref/libpmg_ref.so is the UNMODIFIED reference (/root/reference/proj)
compiled by oracle/Makefile; see oracle/ref_capi.cpp for the wrappers.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libpmg_ref.so")
VARIANT = {"global": 0, "separate": 1, "fused": 2, "boundary": 3}

_lib = None


def available() -> bool:
    return os.path.exists(REF_SO)


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(REF_SO)
        vp, i, i64, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
        pd, pi = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)
        sig = {
            "ref_fill_uniform": (None, [ctypes.c_uint64, i64, vp, i64, vp]),
            "ref_mg_create": (vp, [i, i, i, i, i, i]),
            "ref_mg_destroy": (None, [vp]),
            "ref_mg_create_kind": (vp, [i, i, i, i, i, i, i, pi]),
            "ref_point_gs": (i, [vp, i, vp, vp]),
            "ref_assemble_sparse": (i, [i, i, i, vp, vp, vp, ctypes.POINTER(ctypes.c_int64)]),
            "ref_mg_set_threads": (None, [vp, i]),
            "ref_mg_set_smoothing": (None, [vp, i, i]),
            "ref_mg_set_variant": (None, [vp, i]),
            "ref_mg_total_dofs": (i64, [vp, i]),
            "ref_smooth": (i, [vp, i, i, vp, vp]),
            "ref_apply_laplacian": (i, [vp, i, vp, vp]),
            "ref_residual": (i, [vp, i, vp, vp, vp]),
            "ref_prolongate": (i, [vp, i, vp, vp]),
            "ref_restrict": (i, [vp, i, vp, vp]),
            "ref_vcycle": (i, [vp, i, vp, vp]),
            "ref_compute_rhs": (i, [i, i, i, i, vp]),
            "ref_l2_error_sin": (i, [i, i, i, vp, pd]),
            "ref_l2_error_gen": (i, [i, i, i, vp, pd]),
            "ref_fmg": (i, [vp, i, d, i, vp, pi, vp, i]),
            "ref_gmres": (i, [vp, vp, i, vp, vp, d, i, i, pi, vp, i]),
            "ref_last_history_len": (i, []),
            "ref_gauss_lobatto": (i, [i, vp]),
            "ref_gauss_legendre": (i, [i, vp, vp]),
            "ref_cell_matrices": (i, [i, d, vp, vp]),
            "ref_patch_matrices": (i, [i, d, vp]),
            "ref_fastdiag": (i, [i, i, d, vp, vp, vp]),
            "ref_prolongation_matrix": (i, [i, i, i, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def P(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def fill_uniform(seed: int, n0: int, n1: int):
    """The survey's inputs: std::mt19937_64(seed), U(-1,1), x0 then b."""
    a = np.empty(n0)
    b = np.empty(n1)
    lib().ref_fill_uniform(seed, n0, P(a), n1, P(b))
    return a, b


class RefMg:
    """pmg_ref::MultigridContext<T> (T = double if prec == 0 else float)."""

    def __init__(self, dim, k, L, prec=0, variant="fused", threads=1):
        self.dim, self.k, self.L, self.prec = dim, k, L, prec
        self.dtype = np.float64 if prec == 0 else np.float32
        self.h = ctypes.c_void_p(lib().ref_mg_create(dim, k, L, prec, VARIANT[variant], threads))
        if not self.h.value:
            raise RuntimeError("ref_mg_create failed")

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and _lib is not None:
            _lib.ref_mg_destroy(self.h)

    def set_threads(self, t):
        lib().ref_mg_set_threads(self.h, t)

    def set_smoothing(self, pre, post):
        lib().ref_mg_set_smoothing(self.h, pre, post)

    def set_variant(self, variant):
        lib().ref_mg_set_variant(self.h, VARIANT[variant])

    def n(self, li):
        return lib().ref_mg_total_dofs(self.h, li)

    def _c(self, a):
        return np.ascontiguousarray(a, dtype=self.dtype)

    def smooth(self, li, x, b, variant="fused"):
        x = self._c(x).copy()
        b = self._c(b)
        assert lib().ref_smooth(self.h, li, VARIANT[variant], P(x), P(b)) == 0
        return x

    def apply_laplacian(self, li, x):
        x = self._c(x)
        y = np.zeros_like(x)
        assert lib().ref_apply_laplacian(self.h, li, P(x), P(y)) == 0
        return y

    def residual(self, li, x, b):
        x, b = self._c(x), self._c(b)
        r = np.zeros_like(x)
        assert lib().ref_residual(self.h, li, P(x), P(b), P(r)) == 0
        return r

    def prolongate(self, li_coarse, xc):
        xc = self._c(xc)
        xf = np.zeros(self.n(li_coarse + 1), dtype=self.dtype)
        assert lib().ref_prolongate(self.h, li_coarse, P(xc), P(xf)) == 0
        return xf

    def restrict(self, li_coarse, rf):
        rf = self._c(rf)
        rc = np.zeros(self.n(li_coarse), dtype=self.dtype)
        assert lib().ref_restrict(self.h, li_coarse, P(rf), P(rc)) == 0
        return rc

    def vcycle(self, li, x, b):
        x = self._c(x).copy()
        b = self._c(b)
        assert lib().ref_vcycle(self.h, li, P(x), P(b)) == 0
        return x

    def fmg(self, rhs_kind, tol, max_iterations=100):
        x = np.zeros(self.n(self.L - 1))
        it = ctypes.c_int()
        hist = np.zeros(max_iterations + 2)
        st = lib().ref_fmg(self.h, rhs_kind, tol, max_iterations, P(x), ctypes.byref(it), P(hist), len(hist))
        return st, x, it.value, hist[: it.value + 1].copy()


def gmres(ref64, ref32, mixed, b, tol, restart=30, max_iterations=200):
    """pmg_ref::gmres with the reference's V-cycle preconditioner
    (krylov.cpp:24-171): mixed -> one f32 V-cycle of ref32, else f64 of ref64."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    it = ctypes.c_int()
    hist = np.full(max_iterations + 8, np.nan)
    st = lib().ref_gmres(ref64.h, ref32.h if ref32 is not None else ref64.h, int(mixed), P(b), P(x), tol,
                         restart, max_iterations, ctypes.byref(it), P(hist), len(hist))
    assert st == 0
    return x, it.value, hist[: lib().ref_last_history_len()].copy()


def compute_rhs(dim, k, level, kind):
    n = ((1 << level) * k - 1) ** dim
    b = np.zeros(n)
    assert lib().ref_compute_rhs(dim, k, level, kind, P(b)) == 0
    return b
