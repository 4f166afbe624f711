"""GPU parity at the sizes the performance claims are made on (SURVEY.md §8
configs C2/C3/C4): every smoother organisation the measured dispatch picks
there (vp_point, vp_patch2d, vp_patch3d, vp_smooth_plane, vp_smooth_pp,
vp_smooth) against the reference compiled from /root/reference
(oracle/_ref, all host threads) on the survey's mt19937_64 inputs.

One fused and one boundary smoothing step (smoother.cpp:41-151) and one
residual (multigrid.cpp:268-276) per case; the test also asserts which
kernel organisation ran (pmg_smoother_kernel), so a dispatch change cannot
silently move a claimed kernel out of the tested set.

Tolerances as in test_gpu_parity.py: f64 1e-12 relative, f32 1e-5 (smoother
output relative to ||x_ref||, residual relative to ||b||).

Also: FMG iteration counts identical to the reference for every degree in
2D (L=4) and 3D (L=3) — SURVEY.md §8c's golden 5,3,2,1,1,1,1 for 3D — and the
f32 V-cycle against the residual criterion (1e-5 relative to ||b||).
"""

import os

import numpy as np
import pytest

import refbind

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1
TOL = {np.float64: 1e-12, np.float32: 1e-5}


def rel(a, b):
    nb = np.linalg.norm(np.asarray(b, np.float64))
    return np.linalg.norm(np.asarray(a, np.float64) - np.asarray(b, np.float64)) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def pmg(cuda):
    import paper_2405_19004_b200 as p

    if not refbind.available():
        pytest.fail("oracle/_ref/libpmg_ref.so missing: run __graft_entry__.build() where /root/reference exists")
    return p


# (dim, k, L, dtype, expected kernel of the default dispatch)
LARGE = [
    (3, 2, 6, np.float64, "vp_smooth_plane_kernel"),  # C2, the headline
    (3, 2, 6, np.float32, "vp_smooth_plane_kernel"),
    (3, 1, 9, np.float64, "vp_point_kernel"),  # C3 k=1
    (3, 2, 8, np.float64, "vp_patch3d_kernel"),  # C3 k=2
    (3, 3, 7, np.float64, "vp_smooth_pp_kernel"),  # C3 k=3
    (3, 3, 7, np.float32, "vp_smooth_pp_kernel"),
    (3, 4, 7, np.float64, "vp_smooth_pp_kernel"),  # C3 k=4
    (3, 4, 7, np.float32, "vp_smooth_pp_kernel"),
    (3, 5, 6, np.float64, "vp_smooth_kernel"),  # C3 k=5 (L=6 variant)
    (3, 5, 6, np.float32, "vp_smooth_pp_kernel"),
    (3, 6, 6, np.float64, "vp_smooth_kernel"),  # C3 k=6
    (3, 6, 6, np.float32, "vp_smooth_pp_kernel"),
    (3, 7, 6, np.float64, "vp_smooth_kernel"),  # C3 k=7
    (3, 7, 6, np.float32, "vp_smooth_kernel"),
    (2, 2, 13, np.float64, "vp_patch2d_kernel"),  # C4 k=2
    (2, 3, 12, np.float64, "vp_patch2d_kernel"),  # C4 k=3
    (2, 4, 12, np.float32, "vp_patch2d_kernel"),  # C4 k=4 (f32 dispatch)
    (2, 7, 11, np.float64, "vp_smooth_kernel"),  # C4 k=7
]


@pytest.mark.parametrize("case", LARGE,
                         ids=lambda c: f"d{c[0]}k{c[1]}L{c[2]}{'f64' if c[3] == np.float64 else 'f32'}")
def test_large_smoother_and_residual(pmg, cuda, case):
    dim, k, L, dtype, kernel = case
    ctx = pmg.make_multigrid_context(dim, k, L, dtype=dtype)
    lev = ctx.levels[-1]
    for variant in ("fused", "boundary"):
        got_k = {pmg.smoother_kernel(lev, variant, c) for c in range(1 << dim)}
        assert got_k == {kernel}, (variant, got_k)
    prec = 0 if dtype == np.float64 else 1
    ref = refbind.RefMg(dim, k, L, prec=prec, threads=THREADS)
    n = lev.level.total_dofs
    x0, b = refbind.fill_uniform(42, n, n)
    x0, b = x0.astype(dtype), b.astype(dtype)
    bd = cuda.from_numpy(b).cuda()
    for variant in ("fused", "boundary"):
        xd = cuda.from_numpy(x0.copy()).cuda()
        pmg.smooth(lev, xd, bd, variant)
        want = ref.smooth(L - 1, x0, b, variant)
        err = rel(xd.cpu().numpy(), want)
        assert err < TOL[dtype], (variant, err)
        del want
    r = cuda.empty_like(bd)
    x0d = cuda.from_numpy(x0).cuda()
    pmg.compute_residual(lev, x0d, bd, r)
    want = ref.residual(L - 1, x0, b)
    err = np.linalg.norm(r.cpu().numpy().astype(np.float64) - want) / np.linalg.norm(b.astype(np.float64))
    assert err < TOL[dtype], ("residual", err)
    del ref


# FMG iteration counts, f≡1 and the sine right-hand side, every degree:
# identical to the reference's full_multigrid at a 1e-8 reduction
# (multigrid.cpp:355-400).
FMG = [(3, k, 3) for k in range(1, 8)] + [(2, k, 4) for k in range(1, 8)]


@pytest.mark.parametrize("case", FMG, ids=lambda c: f"d{c[0]}k{c[1]}L{c[2]}")
@pytest.mark.parametrize("rhs", [0, 1], ids=["one", "sin"])
def test_fmg_iteration_counts_all_degrees(pmg, cuda, case, rhs):
    dim, k, L = case
    ref = refbind.RefMg(dim, k, L, threads=THREADS)
    st, xref, it_ref, hist_ref = ref.fmg(rhs, 1e-8)
    assert st == 0
    if dim == 3 and rhs == 0:  # SURVEY.md §8c golden: 3D L=3, f≡1, k=1..7
        assert it_ref == [5, 3, 2, 1, 1, 1, 1][k - 1]
    ctx = pmg.make_multigrid_context(dim, k, L)
    rl = [refbind.compute_rhs(dim, k, lv, rhs) for lv in range(1, L + 1)]
    x = cuda.zeros(ctx.levels[-1].level.total_dofs, dtype=cuda.float64, device="cuda")
    stats = pmg.full_multigrid(ctx, rl, x, 1e-8)
    assert stats.iterations == it_ref
    assert np.allclose(stats.residual_history, hist_ref, rtol=1e-6, atol=1e-9 * hist_ref[0])
    assert rel(x.cpu().numpy(), xref) < 1e-11


# f32 V-cycle: the f64 residual of the GPU iterate and of the reference's
# f32 iterate agree to 1e-5 relative to ||b|| (SURVEY.md §7 "FP32 parity
# definition"), at small sizes and at C2.
@pytest.mark.parametrize("case", [(2, 2, 6), (2, 5, 4), (3, 1, 5), (3, 2, 4), (3, 2, 6), (3, 4, 3), (3, 7, 2)],
                         ids=lambda c: f"d{c[0]}k{c[1]}L{c[2]}")
def test_vcycle_f32_residual_criterion(pmg, cuda, case):
    dim, k, L = case
    ref32 = refbind.RefMg(dim, k, L, prec=1, threads=THREADS)
    ref64 = refbind.RefMg(dim, k, L, prec=0, threads=THREADS)
    ctx = pmg.make_multigrid_context(dim, k, L, dtype=np.float32)
    n = ctx.levels[-1].level.total_dofs
    x0, b = refbind.fill_uniform(42, n, n)
    x0, b = x0.astype(np.float32), b.astype(np.float32)
    want = ref32.vcycle(L - 1, x0, b)
    for use_graph in (False, True):
        xd = cuda.from_numpy(x0.copy()).cuda()
        pmg.v_cycle(ctx, L - 1, xd, cuda.from_numpy(b).cuda(), use_graph=use_graph)
        got = xd.cpu().numpy()
        b64 = b.astype(np.float64)
        r_got = ref64.residual(L - 1, got.astype(np.float64), b64)
        r_want = ref64.residual(L - 1, want.astype(np.float64), b64)
        err = np.linalg.norm(r_got - r_want) / np.linalg.norm(b64)
        assert err < 1e-5, (use_graph, err)


@pytest.mark.parametrize("k,L,dtype,variant", [(2, 6, np.float64, "fused"), (2, 6, np.float32, "boundary"),
                                               (1, 7, np.float64, "fused"), (3, 6, np.float32, "fused"),
                                               (4, 5, np.float64, "fused")])
def test_host_smoother_pipeline_bitwise(cuda, k, L, dtype, variant):
    """pmg_smooth_host runs as an H2D / colour-chunk / D2H pipeline on levels
    of >= 2^20 DoF (capi.cu smooth_host_pipelined): bitwise the device step."""
    import paper_2405_19004_b200 as pmg

    lev = pmg.make_level_context(pmg.build_hierarchy(3, k, L)[-1], dtype=dtype)
    n = lev.level.total_dofs
    assert n >= 1 << 20
    rng = np.random.default_rng(17)
    x0, b = rng.uniform(-1, 1, n).astype(dtype), rng.uniform(-1, 1, n).astype(dtype)
    xd = cuda.from_numpy(x0.copy()).cuda()
    pmg.smooth(lev, xd, cuda.from_numpy(b).cuda(), variant)
    xh = x0.copy()
    pmg.smooth(lev, xh, b, variant)
    assert np.array_equal(xh, xd.cpu().numpy())
    pmg.smooth(lev, xh, b, variant)  # a second step through the same buffers / events
    pmg.smooth(lev, xd, cuda.from_numpy(b).cuda(), variant)
    assert np.array_equal(xh, xd.cpu().numpy())
