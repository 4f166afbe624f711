"""Point Gauss-Seidel smoother and CSR assembly:
assemble_sparse (operator.cpp:194-281), point_gauss_seidel / the sweep
(smoother.cpp:160-166, sparse.cpp:31-47) and the point_gs V-cycle kind
(multigrid.cpp:286-300), each against the reference compiled in oracle/_ref.

CPU: the library's host CSR equals the reference's (structure exactly,
values to 1e-15), and both refuse a level past the 1e7-nonzero budget.
GPU: one device sweep (wavefronts of independent rows in the reference's
lexicographic order) matches the reference's CSR sweep to 1e-12; the point_gs
V-cycle matches ref v_cycle; FMG takes the reference's iteration count."""

import ctypes

import numpy as np
import pytest

import refbind

pytestmark = pytest.mark.skipif(not refbind.available(), reason="oracle/_ref not built")


def ref_csr(dim, k, level):
    lib = refbind.lib()
    nnz = ctypes.c_int64()
    assert lib.ref_assemble_sparse(dim, k, level, None, None, None, ctypes.byref(nnz)) == 0
    m = (1 << level) * k - 1
    rp = np.zeros(m ** dim + 1, dtype=np.int64)
    cols = np.zeros(nnz.value, dtype=np.int32)
    vals = np.zeros(nnz.value)
    assert lib.ref_assemble_sparse(dim, k, level, rp.ctypes.data, cols.ctypes.data, vals.ctypes.data,
                                   ctypes.byref(nnz)) == 0
    return rp, cols, vals


@pytest.mark.parametrize("dim,k,level", [(2, 1, 3), (2, 2, 3), (2, 3, 2), (2, 5, 2), (2, 7, 2),
                                         (3, 1, 3), (3, 2, 2), (3, 3, 2), (3, 4, 1), (3, 6, 1)])
def test_assemble_sparse_matches_reference(dim, k, level):
    import paper_2405_19004_b200 as pmg

    lev = pmg.build_hierarchy(dim, k, level)[-1]
    rp, cols, vals = pmg.assemble_sparse(lev)
    rp_r, cols_r, vals_r = ref_csr(dim, k, level)
    assert np.array_equal(rp, rp_r)
    assert np.array_equal(cols, cols_r)
    np.testing.assert_allclose(vals, vals_r, rtol=1e-14, atol=1e-14 * np.abs(vals_r).max())


def test_assemble_sparse_budget_error():
    import paper_2405_19004_b200 as pmg

    lev = pmg.build_hierarchy(3, 2, 6)[-1]  # ~ 1.3e8 nonzeros > 1e7
    with pytest.raises(RuntimeError, match="budget"):
        pmg.assemble_sparse(lev)
    nnz = ctypes.c_int64()
    assert refbind.lib().ref_assemble_sparse(3, 2, 6, None, None, None, ctypes.byref(nnz)) == 2


def _ref_ctx(dim, k, L, kind):
    st = ctypes.c_int()
    h = refbind.lib().ref_mg_create_kind(dim, k, L, 0, 2, kind, 4, ctypes.byref(st))
    return h, st.value


def test_reference_refuses_f32_point_gs():
    """The behaviour pmg_mg_create_kind mirrors (GPU side: test_point_gs_context_errors)."""
    h, st = _ref_ctx(2, 2, 3, 1)  # f64: fine
    assert h and st == 0
    refbind.lib().ref_mg_destroy(h)
    stf = ctypes.c_int()
    hf = refbind.lib().ref_mg_create_kind(2, 2, 3, 1, 2, 1, 1, ctypes.byref(stf))
    assert not hf and stf.value == 1


@pytest.mark.gpu
@pytest.mark.parametrize("dim,k,level", [(2, 1, 5), (2, 2, 5), (2, 4, 3), (2, 7, 2), (3, 1, 4), (3, 2, 3),
                                         (3, 3, 2), (3, 5, 1)])
def test_point_gs_sweep_vs_reference(cuda, dim, k, level):
    import paper_2405_19004_b200 as pmg

    h, st = _ref_ctx(dim, k, level, 1)
    assert st == 0
    try:
        n = (((1 << level) * k - 1) ** dim)
        rng = np.random.default_rng(7)
        x0, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        xr = x0.copy()
        assert refbind.lib().ref_point_gs(h, level - 1, xr.ctypes.data, b.ctypes.data) == 0
        ctx = pmg.make_level_context(pmg.build_hierarchy(dim, k, level)[-1])
        xd = cuda.from_numpy(x0.copy()).cuda()
        pmg.point_gauss_seidel(ctx, xd, cuda.from_numpy(b).cuda())
        xg = xd.cpu().numpy()
        err = np.abs(xg - xr).max() / np.abs(xr).max()
        assert err < 1e-12, err
        xh = x0.copy()
        pmg.point_gauss_seidel(ctx, xh, b)  # host path
        assert np.array_equal(xh, xg)  # deterministic: fixed lane / front assignment
    finally:
        refbind.lib().ref_mg_destroy(h)


@pytest.mark.gpu
@pytest.mark.parametrize("dim,k,L", [(2, 2, 5), (2, 3, 4), (3, 1, 4), (3, 2, 3), (3, 3, 2)])
def test_point_gs_vcycle_and_fmg_vs_reference(cuda, dim, k, L):
    import paper_2405_19004_b200 as pmg

    h, st = _ref_ctx(dim, k, L, 1)
    assert st == 0
    try:
        mg = pmg.make_multigrid_context(dim, k, L, kind="point_gs")
        n = mg.levels[-1].level.total_dofs
        rng = np.random.default_rng(3)
        x0, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        xr = x0.copy()
        assert refbind.lib().ref_vcycle(h, L - 1, xr.ctypes.data, b.ctypes.data) == 0
        xd = cuda.from_numpy(x0.copy()).cuda()
        pmg.v_cycle(mg, L - 1, xd, cuda.from_numpy(b).cuda())
        err = np.linalg.norm(xd.cpu().numpy() - xr) / np.linalg.norm(xr)
        assert err < 1e-12, err
        # FMG, f = 1, tol 1e-8: identical iteration count
        its = ctypes.c_int()
        hist = np.zeros(64)
        xf = np.zeros(n)
        assert refbind.lib().ref_fmg(h, 0, 1e-8, 50, xf.ctypes.data, ctypes.byref(its), hist.ctypes.data, 64) == 0
        rhs = [pmg.compute_rhs(lev, "one") for lev in pmg.build_hierarchy(dim, k, L)]
        xg = np.zeros(n)
        stats = pmg.full_multigrid(mg, rhs, xg, 1e-8)
        assert stats.iterations == its.value
        np.testing.assert_allclose(stats.residual_history, hist[: its.value + 1], rtol=1e-8, atol=1e-12 * hist[0])
    finally:
        refbind.lib().ref_mg_destroy(h)


@pytest.mark.gpu
def test_point_gs_context_errors(cuda):
    import paper_2405_19004_b200 as pmg

    with pytest.raises(ValueError):
        pmg.make_multigrid_context(2, 2, 3, kind="point_gs", dtype=np.float32)
    with pytest.raises(RuntimeError, match="budget"):
        pmg.make_multigrid_context(3, 2, 6, kind="point_gs")
