"""CPU: pin the numpy oracle (oracle/pmg_oracle.py) before trusting it.

1. SPEC.md known-answer tests (SURVEY.md §4 lists them, all verified on the
   reference during the survey);
2. golden fixtures produced by the reference itself (tests/golden/*.npz,
   made by tests/golden/make_golden.py from oracle/_ref);
3. the SPEC invariants the reference's design calls for (fast-diagonalisation
   identities, transfer adjointness, variant agreement, exact coarse solve).
"""

import glob
import math
import os

import numpy as np
import pytest

from oracle import pmg_oracle as O

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a, np.float64) - np.asarray(b, np.float64)) / (nb if nb else 1.0)


# ---- 1. SPEC known-answer tests ----------------------------------------------


def test_kat_hierarchy_and_numbering():
    lev = O.build_hierarchy(2, 2, 2)[1]
    assert (lev.cells_per_dim, lev.dofs_per_dim, lev.total_dofs) == (4, 7, 49)
    c = O.build_hierarchy(3, 1, 1)[0]
    assert (c.cells_per_dim, c.dofs_per_dim, c.total_dofs) == (2, 1, 1)
    m7 = O.CartesianLevel(2, 2, 2)
    assert O.dof_index(m7, (0, 0)) == 0 and O.dof_index(m7, (3, 2)) == 17
    m5 = O.CartesianLevel(1, 3, 3)  # m = 2*3-1 = 5
    assert O.dof_index(m5, (4, 4, 4)) == 124
    with pytest.raises(ValueError):
        O.build_hierarchy(4, 1, 1)
    with pytest.raises(IndexError):
        O.dof_index(m7, (7, 0))


def test_kat_patch_colours():
    # 2D level 2: 9 patches in 4 colours of sizes {1,2,2,4}
    lev = O.CartesianLevel(2, 2, 1)
    sizes = sorted(
        int(np.prod([len(O._colour_vertices(lev.cells_per_dim, (c >> a) & 1)) for a in range(2)]))
        for c in range(4)
    )
    assert sizes == [1, 2, 2, 4]


def test_kat_element():
    np.testing.assert_allclose(O.gauss_lobatto_points(1), [0, 1])
    np.testing.assert_allclose(O.gauss_lobatto_points(2), [0, 0.5, 1])
    g3 = O.gauss_lobatto_points(3)
    assert abs(g3[1] - 0.27639320225002106) < 1e-15 and abs(g3[2] - 0.72360679774997894) < 1e-15
    m, a = O.cell_matrices_1d(1, 0.25)
    np.testing.assert_allclose(a, [[4, -4], [-4, 4]], rtol=1e-14)
    np.testing.assert_allclose(m, [[1 / 12, 1 / 24], [1 / 24, 1 / 12]], rtol=1e-14)


def test_kat_patch_and_fastdiag():
    pm = O.patch_matrices_1d(1, 0.5)
    np.testing.assert_allclose(pm.stiff_ii, [[4.0]], rtol=1e-14)
    np.testing.assert_allclose(pm.mass_ii, [[1 / 3]], rtol=1e-14)
    np.testing.assert_allclose(pm.stiff_ib, [[-2.0, -2.0]], rtol=1e-14)
    np.testing.assert_allclose(pm.mass_ib, [[1 / 12, 1 / 12]], rtol=1e-14)
    fd = O.make_fastdiag(2, 1, 0.5)  # lambda = 3/h^2 = 12, S = sqrt(3)
    assert abs(fd.eigenvalues[0] - 12.0) < 1e-12 and abs(fd.eigenvectors[0, 0] - math.sqrt(3)) < 1e-12
    # 2D k=1 level-1 patch inverse is r -> 0.375 r
    lc = O.make_level_context(O.CartesianLevel(1, 2, 1))
    x = O.smooth(lc, np.zeros(1), np.array([1.0]))
    assert abs(x[0] - 0.375) < 1e-15
    # assembled 2D k=1 level-1 matrix is [8/3]
    assert abs(O.apply_laplacian(lc, np.array([1.0]))[0] - 8 / 3) < 1e-14


def test_kat_rhs_one():
    lev = O.CartesianLevel(3, 2, 1)  # f = 1, 2D k=1: b_i = h^2
    b = O.compute_rhs(lev, O.f_one)
    np.testing.assert_allclose(b, lev.spacing ** 2, rtol=1e-13)


# ---- 2. golden fixtures produced by the reference ----------------------------


@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: os.path.basename(p)[:-4])
def test_oracle_matches_reference_fixtures(path):
    g = np.load(path)
    dim, k, L, prec = int(g["dim"]), int(g["k"]), int(g["L"]), int(g["prec"])
    dt = np.float64 if prec == 0 else np.float32
    tol = 1e-12 if prec == 0 else 1e-5
    ctx = O.MultigridContext(dim, k, L, dtype=dt)
    lc = ctx.levels[-1]
    x0, b = g["x0"], g["b"]
    for v in O.VARIANTS:
        assert rel(O.smooth(lc, x0, b, v), g[f"smooth_{v}"]) < tol, v
    assert rel(O.apply_laplacian(lc, x0), g["laplacian"]) < tol
    r = O.compute_residual(lc, x0, b)
    assert np.linalg.norm(r - g["residual"]) / np.linalg.norm(b) < tol
    assert rel(O.v_cycle(ctx, L - 1, x0, b), g["vcycle"]) < (1e-11 if prec == 0 else 1e-4)
    if "prolongate" in g:
        assert rel(O.prolongate(ctx.levels[-2], lc, g["xc"]), g["prolongate"]) < tol
        assert rel(O.restrict_vector(ctx.levels[-2], lc, g["rf"]), g["restrict"]) < tol
    for tag in ("one", "sin"):
        key = f"fmg_{tag}_iterations"
        if key in g:
            rhs = [O.compute_rhs(l, O.f_one if tag == "one" else O.f_sin) for l in O.build_hierarchy(dim, k, L)]
            assert rel(rhs[-1], g[f"rhs_{tag}"]) < 1e-12
            x, it, hist = O.full_multigrid(ctx, rhs, 1e-8)
            assert it == int(g[key])
            np.testing.assert_allclose(hist, g[f"fmg_{tag}_history"], rtol=1e-6, atol=1e-9 * hist[0])


def test_survey_golden_norms():
    """C1 norms, reproduced from the stored reference inputs."""
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "c1_2d_q2_l6_f64.npz"))
    assert abs(np.linalg.norm(g["x0"]) - 72.91594658921915) < 1e-10
    ctx = O.MultigridContext(2, 2, 6)
    lc = ctx.levels[-1]
    assert abs(np.linalg.norm(O.compute_residual(lc, g["x0"], g["b"])) - 338.1620349001778) < 1e-9
    x1 = O.smooth(lc, g["x0"], g["b"])
    assert abs(np.linalg.norm(x1) - 43.49331532632719) < 1e-10
    assert abs(np.linalg.norm(O.compute_residual(lc, x1, g["b"])) - 21.67284987997918) < 1e-9
    assert g["fmg_one_iterations"] == 2 and g["fmg_sin_iterations"] == 2


# ---- 3. SPEC invariants --------------------------------------------------------


@pytest.mark.parametrize("k", range(1, 8))
def test_fastdiag_identities(k):
    """S^T M S = I, A S = M S Lambda, lambda > 0."""
    pm = O.patch_matrices_1d(k, 0.125)
    fd = O.make_fastdiag(3, k, 0.125)
    S, lam = fd.eigenvectors, fd.eigenvalues
    np.testing.assert_allclose(S.T @ pm.mass_ii @ S, np.eye(2 * k - 1), atol=1e-12)
    res = pm.stiff_ii @ S - pm.mass_ii @ S @ np.diag(lam)
    assert np.abs(res).max() <= 1e-11 * np.abs(pm.stiff_ii).max()
    assert (lam > 0).all() and (np.diff(lam) > 0).all()


@pytest.mark.parametrize("dim,k", [(2, 1), (2, 3), (2, 5), (3, 1), (3, 2), (3, 4)])
def test_patch_inverse_vs_dense(dim, k):
    """fast-diagonalisation inverse = dense inverse of the
    Kronecker-assembled patch matrix, rel 1e-11."""
    h = 0.25
    pm = O.patch_matrices_1d(k, h)
    fd = O.make_fastdiag(dim, k, h)
    M, A = pm.mass_ii, pm.stiff_ii
    if dim == 2:
        Aj = np.kron(A, M) + np.kron(M, A)
    else:
        Aj = np.kron(np.kron(A, M), M) + np.kron(np.kron(M, A), M) + np.kron(np.kron(M, M), A)
    rng = np.random.default_rng(0)
    r = rng.standard_normal((2 * k - 1,) * dim)
    v = O.apply_patch_inverse(fd, r)
    want = np.linalg.solve(Aj, r.reshape(-1)).reshape(r.shape)
    assert rel(v, want) < 1e-11


@pytest.mark.parametrize("dim,k,L", [(2, 2, 3), (2, 5, 2), (3, 1, 3), (3, 3, 2)])
def test_transfer_adjointness(dim, k, L):
    """<R r, x> = <r, P x>, rel 1e-12."""
    ctx = O.MultigridContext(dim, k, L)
    c, f = ctx.levels[-2], ctx.levels[-1]
    rng = np.random.default_rng(1)
    xc = rng.standard_normal(c.level.total_dofs)
    rf = rng.standard_normal(f.level.total_dofs)
    lhs = np.dot(O.restrict_vector(c, f, rf), xc)
    rhs = np.dot(rf, O.prolongate(c, f, xc))
    assert abs(lhs - rhs) <= 1e-12 * abs(rhs)


@pytest.mark.parametrize("dim,k", [(2, 1), (2, 3), (3, 2), (3, 5)])
def test_level1_exact(dim, k):
    """on level 1 one smoothing step is an exact solve."""
    lc = O.make_level_context(O.CartesianLevel(1, dim, k))
    b = np.random.default_rng(2).standard_normal(lc.level.total_dofs)
    x = O.smooth(lc, np.zeros_like(b), b)
    assert np.linalg.norm(O.compute_residual(lc, x, b)) <= 1e-10 * np.linalg.norm(b)


def test_variant_agreement():
    """all four variants agree to rel 1e-11."""
    lc = O.make_level_context(O.CartesianLevel(3, 2, 3))
    rng = np.random.default_rng(3)
    x, b = rng.standard_normal(lc.level.total_dofs), rng.standard_normal(lc.level.total_dofs)
    outs = [O.smooth(lc, x, b, v) for v in O.VARIANTS]
    for o in outs[1:]:
        assert rel(o, outs[0]) < 1e-11


def test_centro_symmetry_and_parity():
    """The even-odd factorisation of the B200 kernel relies on these: the
    interior rows of the two-cell matrices are centro-symmetric and every
    patch eigenvector is even or odd (reflection symmetry of the patch)."""
    for k in range(1, 8):
        pm = O.patch_matrices_1d(k, 1.0 / 16)
        for B in (pm.mass_if, pm.stiff_if):
            np.testing.assert_allclose(B[::-1, ::-1], B, rtol=0, atol=1e-14 * np.abs(B).max())
        S = O.make_fastdiag(3, k, 1.0 / 16).eigenvectors
        for j in range(2 * k - 1):
            col = S[:, j]
            assert min(np.abs(col[::-1] - col).max(), np.abs(col[::-1] + col).max()) < 1e-10 * np.abs(col).max()
