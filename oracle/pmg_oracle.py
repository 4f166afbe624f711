"""CPU restatement of the reference `pmg` hot path in numpy — TEST INFRASTRUCTURE.

This module is the parity checker for the B200 path. It is imported only by
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline leg; the
product package (`paper_2405_19004_b200`) never imports it and never falls
back to it.

Every function restates one reference function (file:line under
/root/reference/proj) with the same arithmetic, vectorised over all patches of
a colour (patches of one colour have disjoint interiors and read no
same-colour interior, `patches.cpp:11-46`, `SPEC.md:238`, so the vectorised
update equals the reference's sequential/threaded one). It is *pinned* by
tests/test_oracle.py against (1) the SPEC.md known-answer tests, (2) golden
vectors produced by the reference itself compiled from /root/reference
(oracle/_ref, fixtures in tests/golden/ made by tests/golden/make_golden.py)
and (3) the survey's golden norms.

Vector layout is the reference's (`mesh.cpp:42-57`): a flat array of length
N = m^d, direction 0 fastest. Internally a vector is viewed as an array of
shape (m,)*d indexed [i_{d-1}, ..., i_0], i.e. reference direction `a` is numpy
axis d-1-a.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# ---------------------------------------------------------------------------
# mesh  (mesh.hpp:16-27, mesh.cpp:12-57)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class CartesianLevel:
    level: int
    dim: int
    degree: int

    @property
    def cells_per_dim(self) -> int:  # n = 2^l
        return 1 << self.level

    @property
    def dofs_per_dim(self) -> int:  # m = n k - 1
        return self.cells_per_dim * self.degree - 1

    @property
    def spacing(self) -> float:  # h = 1/n
        return 1.0 / self.cells_per_dim

    @property
    def total_dofs(self) -> int:  # N = m^d
        return self.dofs_per_dim ** self.dim


def build_hierarchy(dim: int, degree: int, finest_level: int) -> list[CartesianLevel]:
    """mesh.cpp:12-40 — levels l = 1..L, coarsest has one interior vertex."""
    if dim not in (2, 3):
        raise ValueError("build_hierarchy: dim must be 2 or 3")
    if degree < 1:
        raise ValueError("build_hierarchy: degree must be >= 1")
    if finest_level < 1:
        raise ValueError("build_hierarchy: finest_level must be >= 1")
    return [CartesianLevel(l, dim, degree) for l in range(1, finest_level + 1)]


def dof_index(level: CartesianLevel, multi_index) -> int:
    """mesh.cpp:42-57 — lexicographic, direction 0 contiguous."""
    m = level.dofs_per_dim
    if len(multi_index) != level.dim:
        raise ValueError("dof_index: multi-index size does not match dim")
    idx, stride = 0, 1
    for a in range(level.dim):
        if not 0 <= multi_index[a] < m:
            raise IndexError("dof_index: component out of range")
        idx += multi_index[a] * stride
        stride *= m
    return idx


# ---------------------------------------------------------------------------
# element  (element.cpp)
# ---------------------------------------------------------------------------


def _legendre(n: int, x: float):
    """element.cpp:18-34 — P_n and P_n' on [-1, 1]."""
    if n == 0:
        return 1.0, 0.0
    p0, p1 = 1.0, x
    for j in range(2, n + 1):
        p2 = ((2.0 * j - 1.0) * x * p1 - (j - 1.0) * p0) / j
        p0, p1 = p1, p2
    return p1, n * (x * p1 - p0) / (x * x - 1.0)


def gauss_lobatto_points(k: int) -> np.ndarray:
    """element.cpp:38-78 — Newton on P_k' from Chebyshev guesses, symmetrised."""
    if k < 1:
        raise ValueError("gauss_lobatto_points: degree must be >= 1")
    x = [0.0] * (k + 1)
    x[0], x[k] = -1.0, 1.0
    for i in range(1, k):
        t = math.cos(math.pi * i / k)
        for _ in range(100):
            p, dp = _legendre(k, t)
            d2p = (2.0 * t * dp - k * (k + 1.0) * p) / (1.0 - t * t)
            step = dp / d2p
            t -= step
            if abs(step) < 1e-15:
                break
        x[k - i] = t
    x.sort()
    nodes = [0.5 * (1.0 + v) for v in x]
    for i in range(k // 2 + 1):
        lo = 0.5 * (nodes[i] + 1.0 - nodes[k - i])
        nodes[i] = lo
        nodes[k - i] = 1.0 - lo
    if k % 2 == 0:
        nodes[k // 2] = 0.5
    nodes[0], nodes[k] = 0.0, 1.0
    return np.array(nodes)


def gauss_legendre(q: int):
    """element.cpp:80-125 — q-point rule on [0,1], symmetrised."""
    if q < 1:
        raise ValueError("gauss_legendre: need at least one point")
    xs, ws = [], []
    for i in range(q):
        t = math.cos(math.pi * (i + 0.75) / (q + 0.5))
        for _ in range(100):
            p, dp = _legendre(q, t)
            step = p / dp
            t -= step
            if abs(step) < 1e-15:
                break
        p, dp = _legendre(q, t)
        xs.append(t)
        ws.append(2.0 / ((1.0 - t * t) * dp * dp))
    order = sorted(range(q), key=lambda a: xs[a])
    pts = [0.5 * (1.0 + xs[o]) for o in order]
    wts = [0.5 * ws[o] for o in order]
    for i in range(q // 2):
        p = 0.5 * (pts[i] + 1.0 - pts[q - 1 - i])
        pts[i], pts[q - 1 - i] = p, 1.0 - p
        w = 0.5 * (wts[i] + wts[q - 1 - i])
        wts[i] = wts[q - 1 - i] = w
    if q % 2 == 1:
        pts[q // 2] = 0.5
    return np.array(pts), np.array(wts)


def lagrange_values(nodes, x: float) -> np.ndarray:
    """element.cpp:127-137."""
    n = len(nodes)
    v = np.ones(n)
    for j in range(n):
        for m in range(n):
            if m != j:
                v[j] *= (x - nodes[m]) / (nodes[j] - nodes[m])
    return v


def lagrange_gradients(nodes, x: float) -> np.ndarray:
    """element.cpp:139-154."""
    n = len(nodes)
    g = np.zeros(n)
    for j in range(n):
        for i in range(n):
            if i == j:
                continue
            term = 1.0 / (nodes[j] - nodes[i])
            for m in range(n):
                if m != j and m != i:
                    term *= (x - nodes[m]) / (nodes[j] - nodes[m])
            g[j] += term
    return g


def cell_matrices_1d(k: int, h: float):
    """element.cpp:178-199 — M = h*Mhat, A = Ahat/h with the q = k+1 Gauss rule."""
    if h <= 0.0:
        raise ValueError("cell_matrices_1d: spacing must be positive")
    nodes = gauss_lobatto_points(k)
    pts, wts = gauss_legendre(k + 1)
    n = k + 1
    mass = np.zeros((n, n))
    stiff = np.zeros((n, n))
    for iq in range(n):
        v = lagrange_values(nodes, pts[iq])
        g = lagrange_gradients(nodes, pts[iq])
        w = wts[iq]
        for i in range(n):
            for j in range(n):
                mass[i, j] += h * w * v[i] * v[j]
                stiff[i, j] += (1.0 / h) * w * g[i] * g[j]
    return mass, stiff


def assemble_1d_chain(k: int, h: float, n_cells: int, include_boundary: bool):
    """element.cpp:201-225."""
    cm, ca = cell_matrices_1d(k, h)
    nn = n_cells * k + 1
    mass = np.zeros((nn, nn))
    stiff = np.zeros((nn, nn))
    for c in range(n_cells):
        mass[c * k : c * k + k + 1, c * k : c * k + k + 1] += cm
        stiff[c * k : c * k + k + 1, c * k : c * k + k + 1] += ca
    if include_boundary:
        return mass, stiff
    return mass[1:-1, 1:-1].copy(), stiff[1:-1, 1:-1].copy()


# ---------------------------------------------------------------------------
# fastdiag  (fastdiag.cpp)
# ---------------------------------------------------------------------------


@dataclass
class Patch1DMatrices:
    """fastdiag.hpp:22-31."""

    degree: int
    spacing: float
    mass_full: np.ndarray
    stiff_full: np.ndarray
    mass_ii: np.ndarray
    stiff_ii: np.ndarray
    mass_ib: np.ndarray
    stiff_ib: np.ndarray
    mass_if: np.ndarray
    stiff_if: np.ndarray


def patch_matrices_1d(k: int, h: float) -> Patch1DMatrices:
    """fastdiag.cpp:19-60 — two-cell chain with both endpoints kept."""
    if k < 1:
        raise ValueError("patch_matrices_1d: degree must be >= 1")
    if h <= 0.0:
        raise ValueError("patch_matrices_1d: spacing must be positive")
    mf, af = assemble_1d_chain(k, h, 2, True)
    nc = 2 * k + 1
    ib = [0, nc - 1]
    return Patch1DMatrices(
        k, h, mf, af,
        mf[1:-1, 1:-1].copy(), af[1:-1, 1:-1].copy(),
        mf[1:-1][:, ib].copy(), af[1:-1][:, ib].copy(),
        mf[1:-1, :].copy(), af[1:-1, :].copy(),
    )


def generalized_eigen(a: np.ndarray, m: np.ndarray):
    """fastdiag.cpp:82-121 — A S = M S Lambda via Cholesky reduction (the
    algorithm of LAPACK dsygv itype=1), ascending eigenvalues, M-orthonormal
    eigenvectors, first component of non-negligible magnitude positive."""
    if a.shape != m.shape or a.shape[0] != a.shape[1]:
        raise ValueError("generalized_eigen: matrices must be square, same size")
    ell = np.linalg.cholesky(m)  # raises LinAlgError when M is not SPD
    li = np.linalg.inv(ell)
    c = li @ a @ li.T
    lam, y = np.linalg.eigh(0.5 * (c + c.T))
    s = li.T @ y
    for j in range(s.shape[1]):
        col = s[:, j]
        scale = np.max(np.abs(col))
        sign = 1.0
        for v in col:
            if abs(v) > 1e-12 * scale:
                sign = 1.0 if v > 0 else -1.0
                break
        s[:, j] = sign * col
    return s, lam


@dataclass
class FastDiag:
    """fastdiag.hpp:48-56 (one S/lambda, identical in every direction)."""

    dim: int
    degree: int
    eigenvectors: np.ndarray  # (2k-1)^2
    eigenvalues: np.ndarray  # 2k-1
    inverse_eigen_sums: np.ndarray  # shape (ni,)*dim, axis order [i_{d-1},...,i_0]


def make_fastdiag(dim: int, k: int, h: float) -> FastDiag:
    """fastdiag.cpp:123-159."""
    pm = patch_matrices_1d(k, h)
    s, lam = generalized_eigen(pm.stiff_ii, pm.mass_ii)
    grids = np.meshgrid(*([lam] * dim), indexing="ij")
    total = np.zeros_like(grids[0])
    # sum in direction order a = 0..d-1 (fastdiag.cpp:152-154); numpy axis d-1-a
    for a in range(dim):
        total = total + grids[dim - 1 - a]
    return FastDiag(dim, k, s, lam, 1.0 / total)


def prolongation_matrix(k: int) -> np.ndarray:
    """level_context.cpp:21-34 — (2k+1)x(k+1) two-cell embedding."""
    nodes = gauss_lobatto_points(k)
    p = np.zeros((2 * k + 1, k + 1))
    for f in range(2):
        for t in range(k + 1):
            p[f * k + t, :] = lagrange_values(nodes, 0.5 * (f + nodes[t]))
    return p


@dataclass
class LevelContext:
    """level_context.hpp:17-26."""

    level: CartesianLevel
    cell_mass: np.ndarray
    cell_stiffness: np.ndarray
    patch: Patch1DMatrices
    fastdiag: FastDiag
    prolongation: np.ndarray
    dtype: type = np.float64

    def cast(self, a):
        return np.asarray(a, dtype=self.dtype)


def make_level_context(level: CartesianLevel, dtype=np.float64) -> LevelContext:
    """level_context.cpp:9-36 — setup in f64, cast to T."""
    cm, ca = cell_matrices_1d(level.degree, level.spacing)
    pm = patch_matrices_1d(level.degree, level.spacing)
    fd = make_fastdiag(level.dim, level.degree, level.spacing)
    if dtype != np.float64:
        cast = lambda a: a.astype(dtype)  # noqa: E731
        pm = Patch1DMatrices(pm.degree, pm.spacing, *[cast(getattr(pm, f)) for f in (
            "mass_full", "stiff_full", "mass_ii", "stiff_ii", "mass_ib", "stiff_ib", "mass_if", "stiff_if")])
        fd = FastDiag(fd.dim, fd.degree, cast(fd.eigenvectors), cast(fd.eigenvalues),
                      cast(fd.inverse_eigen_sums))
        cm, ca = cast(cm), cast(ca)
    return LevelContext(level, cm, ca, pm, fd, prolongation_matrix(level.degree).astype(dtype), dtype)


# ---------------------------------------------------------------------------
# tensor contraction helpers (tensor.hpp:27-91)
# ---------------------------------------------------------------------------


def _contract(u: np.ndarray, mat: np.ndarray, direction: int, dim: int) -> np.ndarray:
    """Apply `mat` (rows = output) along reference direction `direction` of the
    trailing `dim` axes of u (which are ordered [t_{d-1},...,t_0])."""
    axis = u.ndim - 1 - direction
    moved = np.moveaxis(u, axis, -1)
    out = moved @ mat.T
    return np.moveaxis(out, -1, axis)


# ---------------------------------------------------------------------------
# patches + smoother (patches.cpp:11-190, smoother.cpp:41-151)
# ---------------------------------------------------------------------------

VARIANTS = ("global", "separate", "fused", "boundary")  # smoother.hpp:21-27


def _colour_vertices(n: int, bit: int) -> np.ndarray:
    """patches.cpp:24-33 — vertices 1..n-1 whose parity is `bit`."""
    return np.arange(1 if bit else 2, n, 2)


def _colour_index_arrays(lev: CartesianLevel, color: int, lo: int, hi: int):
    """Lattice indices (into the zero-ringed vector) of the closure-local
    offsets t in [lo, hi] of every patch of `color`, per direction
    (patches.cpp:71: global node g = k(v-1) - 1 + t, lattice p = g + 1)."""
    k = lev.degree
    out = []
    for a in range(lev.dim):
        v = _colour_vertices(lev.cells_per_dim, (color >> a) & 1)
        t = np.arange(lo, hi + 1)
        out.append(k * (v[:, None] - 1) + t[None, :])
    return out


def _gather(xp: np.ndarray, idx, dim: int) -> np.ndarray:
    """Gather patch tensors from the zero-ringed array xp (shape (m+2,)*dim,
    axes [p_{d-1},...,p_0]) -> shape (P_{d-1},...,P_0, T_{d-1},...,T_0)."""
    sl = []
    for ax in range(dim):  # numpy axis ax <-> direction dim-1-ax
        a = dim - 1 - ax
        shape = [1] * (2 * dim)
        shape[ax] = idx[a].shape[0]
        shape[dim + ax] = idx[a].shape[1]
        sl.append(idx[a].reshape(shape))
    return xp[tuple(sl)]


def _scatter(xp: np.ndarray, idx, dim: int, vals: np.ndarray, mode: str) -> None:
    sl = []
    for ax in range(dim):
        a = dim - 1 - ax
        shape = [1] * (2 * dim)
        shape[ax] = idx[a].shape[0]
        shape[dim + ax] = idx[a].shape[1]
        sl.append(idx[a].reshape(shape))
    key = tuple(np.broadcast_arrays(*sl))
    if mode == "add":
        xp[key] += vals
    else:
        xp[key] = vals


def _pad(lev: CartesianLevel, x: np.ndarray) -> np.ndarray:
    m, d = lev.dofs_per_dim, lev.dim
    xp = np.zeros((m + 2,) * d, dtype=x.dtype)
    xp[(slice(1, m + 1),) * d] = x.reshape((m,) * d)
    return xp


def apply_patch_operator(pm: Patch1DMatrices, dim: int, u: np.ndarray) -> np.ndarray:
    """fastdiag.cpp:199-233 — interior rows of the patch operator, same
    contraction sequence (2D: 4, 3D: 8 contractions, z = M0 u shared)."""
    M, A = pm.mass_if, pm.stiff_if
    if dim == 2:
        z = _contract(u, M, 0, 2)
        r = _contract(z, A, 1, 2)
        z = _contract(u, A, 0, 2)
        r = r + _contract(z, M, 1, 2)
        return r
    z = _contract(u, M, 0, 3)
    t = _contract(z, M, 1, 3)
    r = _contract(t, A, 2, 3)
    t = _contract(z, A, 1, 3)
    r = r + _contract(t, M, 2, 3)
    z = _contract(u, A, 0, 3)
    t2 = _contract(z, M, 1, 3)
    r = r + _contract(t2, M, 2, 3)
    return r


def apply_patch_inverse(fd: FastDiag, r: np.ndarray) -> np.ndarray:
    """fastdiag.cpp:164-192 — (xS) diag(1/sum lambda) (xS^T) r."""
    d = fd.dim
    S = fd.eigenvectors
    t = r
    for a in range(d):
        t = _contract(t, S.T, a, d)
    t = t * fd.inverse_eigen_sums
    for a in range(d):
        t = _contract(t, S, a, d)
    return t


def smooth(ctx: LevelContext, x: np.ndarray, b: np.ndarray, variant: str = "fused") -> np.ndarray:
    """smoother.cpp:41-151 — one colourised multiplicative vertex-patch step.
    Colours in ascending parity code; returns the updated x (new array)."""
    lev = ctx.level
    if x.size != lev.total_dofs or b.size != lev.total_dofs:
        raise ValueError("smooth: vector size does not match level")
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant}")
    d, k = lev.dim, lev.degree
    m = lev.dofs_per_dim
    xp = _pad(lev, np.asarray(x, dtype=ctx.dtype))
    bp = _pad(lev, np.asarray(b, dtype=ctx.dtype))
    for color in range(1 << d):
        if any(len(_colour_vertices(lev.cells_per_dim, (color >> a) & 1)) == 0 for a in range(d)):
            continue
        cl = _colour_index_arrays(lev, color, 0, 2 * k)
        it = _colour_index_arrays(lev, color, 1, 2 * k - 1)
        if variant == "global":
            # smoother.cpp:63-81: r = b - A x once per colour, then local solves
            rg = compute_residual(ctx, xp[(slice(1, m + 1),) * d].reshape(-1), bp[(slice(1, m + 1),) * d].reshape(-1))
            rp = _pad(lev, rg)
            r = _gather(rp, it, d)
        else:
            u = _gather(xp, cl, d)
            bi = _gather(bp, it, d)
            if variant == "boundary":
                # smoother.cpp:128-148: A^{IB} x^B = patch operator with x^I = 0
                inner = (Ellipsis,) + (slice(1, 2 * k),) * d
                u = u.copy()
                u[inner] = 0
            r = bi - apply_patch_operator(ctx.patch, d, u)
        v = apply_patch_inverse(ctx.fastdiag, r)
        _scatter(xp, it, d, v, "replace" if variant == "boundary" else "add")
    return xp[(slice(1, m + 1),) * d].reshape(-1).copy()


def smooth_colour_slab(ctx: LevelContext, x_loc: np.ndarray, b_loc: np.ndarray, color: int, zoff: int,
                       nz_cells: int, vz_lo: int, vz_hi: int) -> None:
    """One colour of the fused smoother (smoother.cpp:109-126) restricted to the
    patches with vertex z in [vz_lo, vz_hi] of a 3D box with the level's n
    cells along x, y and nz_cells along z (a stacked box when nz_cells != n);
    x_loc / b_loc hold the global dof planes z >= zoff. In place on x_loc.
    Checker for the slab decomposition (paper_2405_19004_b200/dd.py)."""
    lev = ctx.level
    assert lev.dim == 3
    k, n, m = lev.degree, lev.cells_per_dim, lev.dofs_per_dim
    nloc = x_loc.size // (m * m)
    if any(len(_colour_vertices(n, (color >> a) & 1)) == 0 for a in range(2)):
        return
    vz = np.array([v for v in range(vz_lo, vz_hi + 1) if v % 2 == ((color >> 2) & 1)], dtype=int)
    if vz.size == 0:
        return
    xp = np.zeros((nloc + 2, m + 2, m + 2), dtype=x_loc.dtype)
    bp = np.zeros_like(xp)
    xp[1:-1, 1:-1, 1:-1] = x_loc.reshape(nloc, m, m)
    bp[1:-1, 1:-1, 1:-1] = b_loc.reshape(nloc, m, m)
    cl = _colour_index_arrays(lev, color, 0, 2 * k)[:2]
    it = _colour_index_arrays(lev, color, 1, 2 * k - 1)[:2]
    # z lattice index p = k (v - 1) + t, local padded plane p - zoff
    cl.append(k * (vz[:, None] - 1) + np.arange(0, 2 * k + 1)[None, :] - zoff)
    it.append(k * (vz[:, None] - 1) + np.arange(1, 2 * k)[None, :] - zoff)
    assert cl[2].min() >= 0 and cl[2].max() <= nloc + 1
    u = _gather(xp, cl, 3)
    bi = _gather(bp, it, 3)
    v = apply_patch_inverse(ctx.fastdiag, bi - apply_patch_operator(ctx.patch, 3, u))
    # write back ONLY the patch interiors (other planes may be in flight)
    _scatter(x_loc.reshape(nloc, m, m), [i - 1 for i in it], 3, v, "add")


# ---------------------------------------------------------------------------
# operator (operator.cpp:122-185, 283-411)
# ---------------------------------------------------------------------------


def _global_1d(lev: CartesianLevel, dtype):
    """Global 1D mass/stiffness over the level with Dirichlet rows/columns
    eliminated (element.cpp:201-225 with include_boundary=false); the level
    matrix is their Kronecker sum (operator.cpp:194-281 relies on the same)."""
    mg, ag = assemble_1d_chain(lev.degree, lev.spacing, lev.cells_per_dim, False)
    return mg.astype(dtype), ag.astype(dtype)


def apply_laplacian(ctx: LevelContext, x: np.ndarray) -> np.ndarray:
    """operator.cpp:122-185 — y = A_l x (sum of d Kronecker terms)."""
    lev = ctx.level
    if x.size != lev.total_dofs:
        raise ValueError("apply_laplacian: vector size does not match level")
    d, m = lev.dim, lev.dofs_per_dim
    # cell matrices in working precision, assembled exactly as the cell loop does
    mg, ag = _global_1d_from_cells(ctx)
    u = np.asarray(x, dtype=ctx.dtype).reshape((m,) * d)
    y = np.zeros_like(u)
    for s in range(d):
        t = u
        for a in range(d):
            t = _contract(t, ag if a == s else mg, a, d)
        y = y + t
    return y.reshape(-1)


def _global_1d_from_cells(ctx: LevelContext):
    lev = ctx.level
    k, n = lev.degree, lev.cells_per_dim
    nn = n * k + 1
    mass = np.zeros((nn, nn), dtype=ctx.dtype)
    stiff = np.zeros((nn, nn), dtype=ctx.dtype)
    for c in range(n):
        mass[c * k : c * k + k + 1, c * k : c * k + k + 1] += ctx.cell_mass
        stiff[c * k : c * k + k + 1, c * k : c * k + k + 1] += ctx.cell_stiffness
    return mass[1:-1, 1:-1], stiff[1:-1, 1:-1]


def compute_residual(ctx: LevelContext, x: np.ndarray, b: np.ndarray) -> np.ndarray:
    """multigrid.cpp:268-276 — r = b - A x."""
    return np.asarray(b, dtype=ctx.dtype) - apply_laplacian(ctx, x)


def vector_norm(v: np.ndarray) -> float:
    """multigrid.cpp:260-266."""
    v = np.asarray(v, dtype=np.float64)
    return float(np.sqrt(np.dot(v, v)))


def f_one(*coords):
    return np.ones(np.broadcast_shapes(*[c.shape for c in coords]))


def f_sin(*coords):
    """-Laplace of u = prod sin(pi x_a)."""
    v = len(coords) * math.pi ** 2
    out = v
    for c in coords:
        out = out * np.sin(math.pi * c)
    return out


def u_sin(*coords):
    out = 1.0
    for c in coords:
        out = out * np.sin(math.pi * c)
    return out


def _cell_points(lev: CartesianLevel, q: int):
    pts, wts = gauss_legendre(q)
    n, h = lev.cells_per_dim, lev.spacing
    xs = ((np.arange(n)[:, None] + pts[None, :]) * h).reshape(-1)
    return pts, wts, xs


def compute_rhs(lev: CartesianLevel, f=f_one) -> np.ndarray:
    """operator.cpp:283-344 — b_i = int f phi_i with q = k+2 Gauss points per
    direction, per cell b_local = (x S^T)(W o F), scatter-added."""
    d, k, n, h = lev.dim, lev.degree, lev.cells_per_dim, lev.spacing
    q = k + 2
    nodes = gauss_lobatto_points(k)
    pts, wts, xs = _cell_points(lev, q)
    shape = np.array([lagrange_values(nodes, p) for p in pts])  # q x (k+1)
    grids = np.meshgrid(*([xs] * d), indexing="ij")  # axis ax <-> direction d-1-ax
    fq = f(*[grids[d - 1 - a] for a in range(d)])
    w1 = np.tile(wts, n)
    wgrid = np.ones_like(fq) * h ** d
    for ax in range(d):
        sh = [1] * d
        sh[ax] = -1
        wgrid = wgrid * w1.reshape(sh)
    fq = fq * wgrid
    # per axis: (n*q) -> (n, k+1) cell-local -> scatter into lattice (n*k+1)
    gath = np.zeros((n * k + 1, n * q))
    for c in range(n):
        gath[c * k : c * k + k + 1, c * q : c * q + q] += shape.T
    t = fq
    for ax in range(d):
        t = np.moveaxis(np.tensordot(gath, t, axes=([1], [ax])), 0, ax)
    t = t[(slice(1, -1),) * d]
    return t.reshape(-1).copy()


def l2_error(lev: CartesianLevel, x: np.ndarray, u_exact=u_sin) -> float:
    """operator.cpp:346-411 — sqrt(sum_cells sum_q w (u_h - u)^2), q = k+2."""
    d, k, n, h = lev.dim, lev.degree, lev.cells_per_dim, lev.spacing
    m = lev.dofs_per_dim
    q = k + 2
    nodes = gauss_lobatto_points(k)
    pts, wts, xs = _cell_points(lev, q)
    shape = np.array([lagrange_values(nodes, p) for p in pts])  # q x (k+1)
    ev = np.zeros((n * q, n * k + 1))
    for c in range(n):
        ev[c * q : c * q + q, c * k : c * k + k + 1] = shape
    xl = np.zeros((n * k + 1,) * d)
    xl[(slice(1, -1),) * d] = np.asarray(x, dtype=np.float64).reshape((m,) * d)
    t = xl
    for ax in range(d):
        t = np.moveaxis(np.tensordot(ev, t, axes=([1], [ax])), 0, ax)
    grids = np.meshgrid(*([xs] * d), indexing="ij")
    e = t - u_exact(*[grids[d - 1 - a] for a in range(d)])
    w1 = np.tile(wts, n)
    wgrid = np.ones_like(e) * h ** d
    for ax in range(d):
        sh = [1] * d
        sh[ax] = -1
        wgrid = wgrid * w1.reshape(sh)
    return float(np.sqrt(np.sum(wgrid * e * e)))


# ---------------------------------------------------------------------------
# multigrid (multigrid.cpp:71-400)
# ---------------------------------------------------------------------------


def prolongation_1d_global(coarse: CartesianLevel, p: np.ndarray) -> np.ndarray:
    """The 1D factor of prolongate (multigrid.cpp:71-160): fine lattice node
    p_f is owned by coarse cell c with r = p_f - 2ck in [1, 2k] (the r_a >= 1
    rule of :129-158) and gets sum_t P[r][t] x_c[ck + t]; boundary nodes drop."""
    k = coarse.degree
    nc, nf = coarse.cells_per_dim, 2 * coarse.cells_per_dim
    mc, mf = nc * k - 1, nf * k - 1
    pg = np.zeros((mf, mc), dtype=p.dtype)
    for pf in range(1, nf * k):
        c = (pf - 1) // (2 * k)
        r = pf - 2 * c * k
        for t in range(k + 1):
            qc = c * k + t
            if 1 <= qc <= nc * k - 1:
                pg[pf - 1, qc - 1] = p[r, t]
    return pg


def prolongate(coarse: LevelContext, fine: LevelContext, xc: np.ndarray) -> np.ndarray:
    """multigrid.cpp:71-160 — exact embedding, as a Kronecker product of the 1D
    global factor (same per-cell arithmetic up to summation order)."""
    cl = coarse.level
    d = cl.dim
    pg = prolongation_1d_global(cl, fine.prolongation)
    t = np.asarray(xc, dtype=fine.dtype).reshape((cl.dofs_per_dim,) * d)
    for a in range(d):
        t = _contract(t, pg, a, d)
    return t.reshape(-1)


def restrict_vector(coarse: LevelContext, fine: LevelContext, rf: np.ndarray) -> np.ndarray:
    """multigrid.cpp:162-248 — exact transpose of prolongate."""
    cl, fl = coarse.level, fine.level
    d = cl.dim
    pg = prolongation_1d_global(cl, fine.prolongation)
    t = np.asarray(rf, dtype=fine.dtype).reshape((fl.dofs_per_dim,) * d)
    for a in range(d):
        t = _contract(t, pg.T, a, d)
    return t.reshape(-1)


class MultigridContext:
    """multigrid.hpp:34-49."""

    def __init__(self, dim, degree, finest_level, variant="fused", dtype=np.float64):
        self.levels = [make_level_context(l, dtype) for l in build_hierarchy(dim, degree, finest_level)]
        self.variant = variant
        self.pre_smooth = 1
        self.post_smooth = 1
        self.dtype = dtype


def coarse_solve(ctx: MultigridContext, b: np.ndarray) -> np.ndarray:
    """multigrid.cpp:304-309 — zero start, one fused smooth on index 0."""
    lc = ctx.levels[0]
    return smooth(lc, np.zeros(lc.level.total_dofs, dtype=ctx.dtype), b, "fused")


def v_cycle(ctx: MultigridContext, li: int, x: np.ndarray, b: np.ndarray) -> np.ndarray:
    """multigrid.cpp:313-348 — Alg. 1 with pre/post = 1."""
    if li == 0:
        return coarse_solve(ctx, b)
    lev = ctx.levels[li]
    x = np.asarray(x, dtype=ctx.dtype).copy()
    for _ in range(ctx.pre_smooth):
        x = smooth(lev, x, b, ctx.variant)
    r = compute_residual(lev, x, b)
    bc = restrict_vector(ctx.levels[li - 1], lev, r)
    xc = v_cycle(ctx, li - 1, np.zeros_like(bc), bc)
    x = x + prolongate(ctx.levels[li - 1], lev, xc)
    for _ in range(ctx.post_smooth):
        x = smooth(lev, x, b, ctx.variant)
    return x


def full_multigrid(ctx: MultigridContext, rhs_per_level, tol: float, max_iterations: int = 100):
    """multigrid.cpp:355-400 — nested iteration, then V-cycles until
    ||b - A x|| <= tol ||b||. Returns (x, iterations, history)."""
    if tol <= 0.0:
        raise ValueError("full_multigrid: tol must be positive")
    L = len(ctx.levels) - 1
    x = coarse_solve(ctx, rhs_per_level[0])
    for li in range(1, L + 1):
        x = prolongate(ctx.levels[li - 1], ctx.levels[li], x)
        x = v_cycle(ctx, li, x, rhs_per_level[li])
    bL = rhs_per_level[L]
    delta0 = vector_norm(bL)
    hist = [delta0]
    delta = delta0
    it = 0
    while delta > tol * delta0:
        if it >= max_iterations:
            raise RuntimeError("full_multigrid: no convergence")
        x = v_cycle(ctx, L, x, bL)
        delta = vector_norm(compute_residual(ctx.levels[L], x, bL))
        hist.append(delta)
        it += 1
    return x, it, hist


# ---------------------------------------------------------------------------
# algorithmic cost model — used by bench.py for roofline
# ---------------------------------------------------------------------------


def smoother_flops_per_patch(dim: int, k: int) -> int:
    """Reference contraction sequence flops (fastdiag.cpp:199-233, 164-192,
    smoother.cpp:119-120, patches.cpp:119)."""
    ni, nc = 2 * k - 1, 2 * k + 1
    if dim == 3:
        return 4 * ni * nc ** 3 + 6 * ni ** 2 * nc ** 2 + 6 * ni ** 3 * nc + 12 * ni ** 4 + 3 * ni ** 3
    return 4 * ni * nc ** 2 + 4 * ni ** 2 * nc + 8 * ni ** 3 + 3 * ni ** 2
