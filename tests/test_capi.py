"""CPU: the C-ABI library loads, exports every symbol include/pmg_b200.h
declares, its host setup matches the reference's setup, and its error
behaviour mirrors the reference's exceptions. No GPU compute here."""

import ctypes
import os
import re

import numpy as np
import pytest

import refbind
from oracle import pmg_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pmg_b200.h")


@pytest.fixture(scope="module")
def lib():
    import paper_2405_19004_b200 as pmg

    return pmg.load()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pmg_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(lib):
    names = declared_functions()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/pmg_b200.h but not exported"


def test_python_binding_covers_header():
    from paper_2405_19004_b200 import _lib

    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert set(declared_functions()) <= bound


def host_setup(lib, dim, k, level):
    ni, nc = 2 * k - 1, 2 * k + 1
    out = {"S": np.zeros((ni, ni)), "lambda": np.zeros(ni), "mass_if": np.zeros((ni, nc)),
           "stiff_if": np.zeros((ni, nc)), "prolongation": np.zeros((nc, k + 1)),
           "cell_mass": np.zeros((k + 1, k + 1)), "cell_stiffness": np.zeros((k + 1, k + 1)),
           "band_mass": np.zeros((k, 2 * k + 1)), "band_stiff": np.zeros((k, 2 * k + 1))}
    perm = np.zeros(ni, dtype=np.int32)
    P = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
    st = lib.pmg_host_level_setup(dim, k, level, P(out["S"]), P(out["lambda"]), P(out["mass_if"]),
                                  P(out["stiff_if"]), P(out["prolongation"]), P(out["cell_mass"]),
                                  P(out["cell_stiffness"]), P(out["band_mass"]), P(out["band_stiff"]),
                                  perm.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
    assert st == 0
    out["perm"] = perm
    return out


@pytest.mark.parametrize("k", range(1, 8))
def test_host_setup_matches_reference(lib, k):
    """Setup (element.cpp, fastdiag.cpp, level_context.cpp) vs the reference's
    own numbers from oracle/_ref (LAPACK dsygv there, Jacobi here)."""
    level = 3
    h = 1.0 / (1 << level)
    s = host_setup(lib, 3, k, level)
    ni, nc = 2 * k - 1, 2 * k + 1
    if refbind.available():
        R = refbind.lib()
        pm = np.zeros(2 * nc * nc + 2 * ni * ni + 4 * ni + 2 * ni * nc)
        assert R.ref_patch_matrices(k, h, refbind.P(pm)) == 0
        off = 2 * nc * nc + 2 * ni * ni + 4 * ni
        mif, aif = pm[off:off + ni * nc].reshape(ni, nc), pm[off + ni * nc:].reshape(ni, nc)
        S, lam, inv = np.zeros((ni, ni)), np.zeros(ni), np.zeros(ni ** 3)
        assert R.ref_fastdiag(3, k, h, refbind.P(S), refbind.P(lam), refbind.P(inv)) == 0
        P_ = np.zeros((nc, k + 1))
        assert R.ref_prolongation_matrix(3, k, level, refbind.P(P_)) == 0
        cm, ca = np.zeros((k + 1, k + 1)), np.zeros((k + 1, k + 1))
        assert R.ref_cell_matrices(k, h, refbind.P(cm), refbind.P(ca)) == 0
    else:
        pmo = O.patch_matrices_1d(k, h)
        mif, aif = pmo.mass_if, pmo.stiff_if
        fd = O.make_fastdiag(3, k, h)
        S, lam = fd.eigenvectors, fd.eigenvalues
        P_ = O.prolongation_matrix(k)
        cm, ca = O.cell_matrices_1d(k, h)
    np.testing.assert_allclose(s["mass_if"], mif, rtol=0, atol=1e-14 * np.abs(mif).max())
    np.testing.assert_allclose(s["stiff_if"], aif, rtol=0, atol=1e-13 * np.abs(aif).max())
    np.testing.assert_allclose(s["lambda"], lam, rtol=1e-12)
    np.testing.assert_allclose(s["S"], S, rtol=0, atol=1e-11 * np.abs(S).max())
    np.testing.assert_allclose(s["prolongation"], P_, rtol=0, atol=1e-14)
    np.testing.assert_allclose(s["cell_mass"], cm, rtol=0, atol=1e-14 * np.abs(cm).max())
    np.testing.assert_allclose(s["cell_stiffness"], ca, rtol=0, atol=1e-13 * np.abs(ca).max())


@pytest.mark.parametrize("k", range(1, 8))
def test_band_rows_reassemble_global_operator(lib, k):
    """The device level operator's banded 1D rows are exactly the assembled
    global 1D matrices (element.cpp:201-225, include_boundary=false)."""
    level = 3
    s = host_setup(lib, 2, k, level)
    n = 1 << level
    mg, ag = O.assemble_1d_chain(k, 1.0 / n, n, False)
    m = n * k - 1
    for band, G in ((s["band_mass"], mg), (s["band_stiff"], ag)):
        R = np.zeros((m, m))
        for p in range(1, m + 1):
            r = p % k
            for o in range(2 * k + 1):
                q = p - k + o
                if 1 <= q <= m:
                    R[p - 1, q - 1] = band[r, o]
        np.testing.assert_allclose(R, G, rtol=0, atol=1e-13 * np.abs(G).max())


@pytest.mark.parametrize("k", range(1, 8))
def test_even_odd_mode_order(lib, k):
    """Modes reordered even-first: K even eigenvectors, then K-1 odd ones."""
    s = host_setup(lib, 3, k, 3)
    S, perm = s["S"], s["perm"]
    assert sorted(perm.tolist()) == list(range(2 * k - 1))
    for c, j in enumerate(perm):
        col = S[:, j]
        sign = 1.0 if c < k else -1.0
        np.testing.assert_allclose(col[::-1], sign * col, atol=1e-10 * np.abs(col).max())


@pytest.mark.parametrize("dim,k,level", [(2, 1, 3), (2, 3, 3), (3, 2, 2), (3, 4, 2)])
@pytest.mark.parametrize("kind", [0, 1])
def test_host_rhs_and_l2(lib, dim, k, level, kind):
    """compute_rhs (operator.cpp:283-344) and l2_error (:346-411) on the host."""
    n = ((1 << level) * k - 1) ** dim
    b = np.zeros(n)
    assert lib.pmg_compute_rhs_host(dim, k, level, kind, b.ctypes.data_as(ctypes.POINTER(ctypes.c_double))) == 0
    want = refbind.compute_rhs(dim, k, level, kind) if refbind.available() else \
        O.compute_rhs(O.CartesianLevel(level, dim, k), O.f_one if kind == 0 else O.f_sin)
    assert np.linalg.norm(b - want) <= 1e-12 * np.linalg.norm(want)
    x = np.random.default_rng(5).standard_normal(n)
    e = ctypes.c_double()
    assert lib.pmg_l2_error_sin_host(dim, k, level, x.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                     ctypes.byref(e)) == 0
    assert abs(e.value - O.l2_error(O.CartesianLevel(level, dim, k), x)) <= 1e-12 * e.value


def test_errors_mirror_reference(lib):
    import paper_2405_19004_b200 as pmg

    ni = np.zeros(1)
    P = ctypes.POINTER(ctypes.c_double)
    # invalid arguments -> PMG_ERR_INVALID (std::invalid_argument in the reference)
    assert lib.pmg_host_level_setup(4, 1, 1, *([None] * 9), None) == 1
    assert lib.pmg_host_level_setup(3, 0, 1, *([None] * 9), None) == 1
    assert lib.pmg_compute_rhs_host(5, 1, 1, 0, ni.ctypes.data_as(P)) == 1
    assert b"dim" in lib.pmg_last_error()
    with pytest.raises(ValueError):
        pmg.build_hierarchy(4, 1, 1)
    with pytest.raises(ValueError):
        pmg.make_multigrid_context(3, 2, 0)
    with pytest.raises(ValueError):
        pmg.make_multigrid_context(3, 2, 2, kind="bogus")


def test_no_cpu_fallback_without_gpu(lib):
    """The product path fails loudly instead of computing on the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_2405_19004_b200 as pmg

    with pytest.raises(RuntimeError):
        pmg.make_level_context(pmg.CartesianLevel(2, 3, 2))
    h = ctypes.c_void_p()
    assert lib.pmg_mg_create(3, 2, 2, 0, 2, 0, ctypes.byref(h)) in (2, 4)


def test_smoother_impl_switch(lib):
    import paper_2405_19004_b200 as pmg

    assert lib.pmg_set_smoother_impl(7) != 0
    assert lib.pmg_set_smoother_impl(-1) != 0
    try:
        for name in ["line", "plane", "sweep", "patch", "auto"]:
            pmg.set_smoother_impl(name)
            assert pmg.get_smoother_impl() == name
        with pytest.raises(ValueError):
            pmg.set_smoother_impl("tensor")
    finally:
        pmg.set_smoother_impl("auto")
