"""GPU parity: the CUDA path (through the C-ABI) against the reference
library compiled from /root/reference (oracle/_ref) on the same seeded inputs.

Tolerances (BASELINE.json north star): f64 relative 1e-12 on smoother output,
operator/residual, transfers and V-cycle; f32 relative 1e-5 (residuals
relative to ||b||, SURVEY.md §7 "FP32 parity definition"); FMG iteration
counts identical at a 1e-8 reduction.
"""

import ctypes

import numpy as np
import pytest

import refbind

pytestmark = pytest.mark.gpu

TOL = {np.float64: 1e-12, np.float32: 1e-5}

# (dim, degree, finest level): every degree 1..7 in 2D and 3D at sizes the
# reference finishes in well under a second
CASES = [
    (2, 1, 5), (2, 2, 6), (2, 3, 4), (2, 4, 4), (2, 5, 3), (2, 6, 3), (2, 7, 3),
    (3, 1, 4), (3, 2, 4), (3, 3, 3), (3, 4, 3), (3, 5, 2), (3, 6, 2), (3, 7, 2),
]


def ctypes_double():
    return ctypes.c_double()


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a, np.float64) - np.asarray(b, np.float64)) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def pmg(cuda):
    import paper_2405_19004_b200 as p

    if not refbind.available():
        pytest.fail("oracle/_ref/libpmg_ref.so missing: run __graft_entry__.build() where /root/reference exists")
    return p


def inputs(n, dtype, seed=42):
    x, b = refbind.fill_uniform(seed, n, n)
    return x.astype(dtype), b.astype(dtype)


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"d{c[0]}k{c[1]}L{c[2]}")
def test_smoother_variants(pmg, cuda, case, dtype):
    dim, k, L = case
    ref = refbind.RefMg(dim, k, L, prec=0 if dtype == np.float64 else 1)
    ctx = pmg.make_multigrid_context(dim, k, L, dtype=dtype)
    lev = ctx.levels[-1]
    x0, b = inputs(lev.level.total_dofs, dtype)
    want = ref.smooth(L - 1, x0, b, "fused")
    for variant in ["fused", "boundary", "separate", "global", "naive"]:
        xd = dev(cuda, x0.copy())
        pmg.smooth(lev, xd, dev(cuda, b), variant)
        got = xd.cpu().numpy()
        assert rel(got, want) < TOL[dtype], (variant, rel(got, want))
        if variant != "naive":
            want_v = ref.smooth(L - 1, x0, b, variant)
            assert rel(got, want_v) < TOL[dtype], (variant, rel(got, want_v))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"d{c[0]}k{c[1]}L{c[2]}")
def test_operator_and_residual(pmg, cuda, case, dtype):
    dim, k, L = case
    ref = refbind.RefMg(dim, k, L, prec=0 if dtype == np.float64 else 1)
    ctx = pmg.make_multigrid_context(dim, k, L, dtype=dtype)
    lev = ctx.levels[-1]
    x0, b = inputs(lev.level.total_dofs, dtype)
    y = cuda.zeros_like(dev(cuda, x0))
    pmg.apply_laplacian(lev, dev(cuda, x0), y)
    want = ref.apply_laplacian(L - 1, x0)
    assert rel(y.cpu().numpy(), want) < TOL[dtype]
    r = cuda.zeros_like(y)
    pmg.compute_residual(lev, dev(cuda, x0), dev(cuda, b), r)
    want = ref.residual(L - 1, x0, b)
    err = np.linalg.norm(r.cpu().numpy().astype(np.float64) - want) / np.linalg.norm(b.astype(np.float64))
    assert err < TOL[dtype]
    if dtype == np.float64:
        assert rel(r.cpu().numpy(), want) < 1e-12


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"d{c[0]}k{c[1]}L{c[2]}")
def test_transfers(pmg, cuda, case, dtype):
    dim, k, L = case
    if L < 2:
        pytest.skip("needs two levels")
    ref = refbind.RefMg(dim, k, L, prec=0 if dtype == np.float64 else 1)
    ctx = pmg.make_multigrid_context(dim, k, L, dtype=dtype)
    c, f = ctx.levels[-2], ctx.levels[-1]
    xc, _ = inputs(c.level.total_dofs, dtype, seed=7)
    rf, _ = inputs(f.level.total_dofs, dtype, seed=9)
    xf = cuda.zeros(f.level.total_dofs, dtype=cuda.float64 if dtype == np.float64 else cuda.float32, device="cuda")
    pmg.prolongate(c, f, dev(cuda, xc), xf)
    assert rel(xf.cpu().numpy(), ref.prolongate(L - 2, xc)) < TOL[dtype]
    rc = cuda.zeros(c.level.total_dofs, dtype=xf.dtype, device="cuda")
    pmg.restrict_vector(c, f, dev(cuda, rf), rc)
    assert rel(rc.cpu().numpy(), ref.restrict(L - 2, rf)) < TOL[dtype]
    # accumulate form used by the V-cycle: x += P xc
    base = dev(cuda, rf.copy())
    pmg.prolongate(c, f, dev(cuda, xc), base, accumulate=True)
    assert rel(base.cpu().numpy(), rf.astype(np.float64) + ref.prolongate(L - 2, xc)) < TOL[dtype]


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"d{c[0]}k{c[1]}L{c[2]}")
def test_vcycle(pmg, cuda, case, dtype):
    dim, k, L = case
    ref = refbind.RefMg(dim, k, L, prec=0 if dtype == np.float64 else 1)
    ctx = pmg.make_multigrid_context(dim, k, L, dtype=dtype)
    lev = ctx.levels[-1]
    x0, b = inputs(lev.level.total_dofs, dtype)
    want = ref.vcycle(L - 1, x0, b)
    for use_graph in (False, True):
        xd = dev(cuda, x0.copy())
        pmg.v_cycle(ctx, L - 1, xd, dev(cuda, b), use_graph=use_graph)
        assert rel(xd.cpu().numpy(), want) < (1e-11 if dtype == np.float64 else 1e-4)


@pytest.mark.parametrize("case", [(2, 1, 4), (2, 2, 6), (2, 3, 4), (3, 1, 4), (3, 2, 4), (3, 3, 3), (3, 4, 3)],
                         ids=lambda c: f"d{c[0]}k{c[1]}L{c[2]}")
@pytest.mark.parametrize("rhs", [0, 1], ids=["one", "sin"])
def test_fmg_iteration_counts(pmg, cuda, case, rhs):
    dim, k, L = case
    ref = refbind.RefMg(dim, k, L)
    st, xref, it_ref, hist_ref = ref.fmg(rhs, 1e-8)
    assert st == 0
    ctx = pmg.make_multigrid_context(dim, k, L)
    rl = [refbind.compute_rhs(dim, k, l, rhs) for l in range(1, L + 1)]
    x = cuda.zeros(ctx.levels[-1].level.total_dofs, dtype=cuda.float64, device="cuda")
    stats = pmg.full_multigrid(ctx, rl, x, 1e-8)
    assert stats.iterations == it_ref
    # histories agree to rounding; entries near machine precision relative to ||b||
    assert np.allclose(stats.residual_history, hist_ref, rtol=1e-6, atol=1e-9 * hist_ref[0])
    assert rel(x.cpu().numpy(), xref) < 1e-11


@pytest.mark.parametrize("dim,k", [(2, 1), (2, 4), (3, 2), (3, 7)])
def test_level1_exact_solve(pmg, cuda, dim, k):
    """on level 1 one smoothing step solves A x = b exactly."""
    ctx = pmg.make_multigrid_context(dim, k, 1)
    lev = ctx.levels[0]
    n = lev.level.total_dofs
    _, b = inputs(n, np.float64)
    x = cuda.zeros(n, dtype=cuda.float64, device="cuda")
    bd = dev(cuda, b)
    pmg.smooth(lev, x, bd)
    r = cuda.zeros_like(x)
    pmg.compute_residual(lev, x, bd, r)
    assert r.norm().item() <= 1e-10 * np.linalg.norm(b)


def test_survey_goldens(pmg, cuda):
    """SURVEY.md §8c golden norms for C1 (2D Q2 L=6), mt19937_64(42) inputs."""
    ctx = pmg.make_multigrid_context(2, 2, 6)
    lev = ctx.levels[-1]
    x0, b = inputs(lev.level.total_dofs, np.float64)
    assert abs(np.linalg.norm(x0) - 72.91594658921915) < 1e-10
    xd, bd = dev(cuda, x0.copy()), dev(cuda, b)
    r = cuda.zeros_like(xd)
    pmg.compute_residual(lev, xd, bd, r)
    assert abs(r.norm().item() - 338.1620349001778) < 1e-9
    pmg.smooth(lev, xd, bd)
    assert abs(xd.norm().item() - 43.49331532632719) < 1e-10
    pmg.compute_residual(lev, xd, bd, r)
    assert abs(r.norm().item() - 21.67284987997918) < 1e-9
    xd = dev(cuda, x0.copy())
    pmg.v_cycle(ctx, 5, xd, bd)
    assert abs(xd.norm().item() - 783.2195575549429) < 1e-8
    pmg.compute_residual(lev, xd, bd, r)
    assert abs(r.norm().item() - 0.7452650912722393) < 1e-9


def test_host_buffer_entry_points(pmg, cuda):
    """numpy (host) vectors go through the *_host C-ABI calls (H2D, kernel, D2H)."""
    dim, k, L = 3, 3, 3
    ref = refbind.RefMg(dim, k, L)
    ctx = pmg.make_multigrid_context(dim, k, L)
    lev = ctx.levels[-1]
    x0, b = inputs(lev.level.total_dofs, np.float64)
    x = x0.copy()
    pmg.smooth(lev, x, b)
    assert rel(x, ref.smooth(L - 1, x0, b)) < 1e-12
    y = np.zeros_like(x0)
    pmg.apply_laplacian(lev, x0, y)
    assert rel(y, ref.apply_laplacian(L - 1, x0)) < 1e-12
    x = x0.copy()
    pmg.v_cycle(ctx, L - 1, x, b)
    assert rel(x, ref.vcycle(L - 1, x0, b)) < 1e-11


def test_determinism(pmg, cuda):
    """No atomics anywhere: two runs are bitwise identical."""
    ctx = pmg.make_multigrid_context(3, 4, 3)
    lev = ctx.levels[-1]
    x0, b = inputs(lev.level.total_dofs, np.float64)
    outs = []
    for _ in range(2):
        xd = dev(cuda, x0.copy())
        pmg.v_cycle(ctx, 2, xd, dev(cuda, b))
        outs.append(xd.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("world,k,level,stack", [(2, 2, 4, 1), (4, 3, 3, 1), (3, 1, 5, 1), (8, 2, 4, 1),
                                                 (2, 4, 3, 2), (4, 2, 3, 4)])
def test_slab_decomposition_virtual_ranks(pmg, cuda, world, k, level, stack):
    """P slabs (virtual ranks on one GPU, plane copies in place
    of NCCL) give BITWISE the single-domain GPU result; for the unit cube that
    is also the reference's smooth."""
    from paper_2405_19004_b200 import dd

    ctx = pmg.make_multigrid_context(3, k, level)
    lev = ctx.levels[-1]
    full = dd.make_plan(1, 0, k, level, stack)
    n = full.nplanes * full.plane_size
    x0, b = refbind.fill_uniform(42, n, n)
    xg, bg = dev(cuda, x0.copy()), dev(cuda, b)
    dd.virtual_smooth([full], [dd.gpu_kernel(lev, full, xg, bg)], [xg])
    ps = [dd.make_plan(world, r, k, level, stack) for r in range(world)]
    xs = [dd.scatter_global(p, dev(cuda, x0)).clone() for p in ps]
    bs = [dd.scatter_global(p, bg).clone() for p in ps]
    dd.virtual_smooth(ps, [dd.gpu_kernel(lev, p, x, bb) for p, x, bb in zip(ps, xs, bs)], xs)
    got = cuda.cat([dd.owned_part(p, x) for p, x in zip(ps, xs)])
    assert cuda.equal(got, xg)
    if stack == 1:
        xs1 = dev(cuda, x0.copy())
        pmg.smooth(lev, xs1, bg)
        assert cuda.equal(xs1, xg)
        ref = refbind.RefMg(3, k, level)
        assert rel(xg.cpu().numpy(), ref.smooth(level - 1, x0, b)) < 1e-12


def test_cpp_shim(pmg, cuda):
    """C++ host code (include/pmg_b200.hpp over the C-ABI) vs the reference."""
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(__file__), "cpp", "_bin", "shim_parity")
    if not os.path.exists(exe):
        pytest.fail("tests/cpp/_bin/shim_parity missing: run __graft_entry__.build()")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK" in out.stdout


# Both kernel organisations of the 3D low-degree smoother (line-per-thread and
# plane-streaming) against the reference, including levels whose colour sizes
# are not multiples of the patches-per-CTA (ragged last CTA) and level 1
# (a single patch, the coarse solve).
@pytest.mark.parametrize("impl", ["auto", "line", "plane", "sweep", "patch"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("case", [(2, 1, 1), (2, 1, 6), (2, 2, 1), (2, 2, 3), (2, 2, 6), (2, 3, 1), (2, 3, 5), (3, 1, 1), (3, 1, 5), (3, 2, 1), (3, 2, 3), (3, 2, 5), (3, 3, 1), (3, 3, 4)],
                         ids=lambda c: f"d{c[0]}k{c[1]}L{c[2]}")
def test_smoother_impls(pmg, cuda, case, dtype, impl):
    dim, k, L = case
    ref = refbind.RefMg(dim, k, L, prec=0 if dtype == np.float64 else 1)
    ctx = pmg.make_multigrid_context(dim, k, L, dtype=dtype)
    lev = ctx.levels[-1]
    x0, b = inputs(lev.level.total_dofs, dtype, seed=7)
    pmg.set_smoother_impl(impl)
    try:
        for variant in ["fused", "boundary"]:
            xd = dev(cuda, x0.copy())
            pmg.smooth(lev, xd, dev(cuda, b), variant)
            want = ref.smooth(L - 1, x0, b, variant)
            assert rel(xd.cpu().numpy(), want) < TOL[dtype], (variant, rel(xd.cpu().numpy(), want))
    finally:
        pmg.set_smoother_impl("auto")


# The persistent all-colour sweep must reproduce the per-colour launches
# bitwise (same per-patch arithmetic, same colour order), over several steps
# (the counters are reset by the last CTA of each launch) and inside a
# graph-captured V-cycle.
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("L", [2, 3, 4, 5])
def test_sweep_bitwise(pmg, cuda, L, dtype):
    dim, k = 3, 2
    ctx = pmg.make_multigrid_context(dim, k, L, dtype=dtype)
    lev = ctx.levels[-1]
    x0, b = inputs(lev.level.total_dofs, dtype, seed=11)
    out = {}
    try:
        for impl in ["plane", "sweep"]:
            pmg.set_smoother_impl(impl)
            xd = dev(cuda, x0.copy())
            bd = dev(cuda, b)
            for _ in range(3):
                for variant in ["fused", "boundary"]:
                    pmg.smooth(lev, xd, bd, variant)
            xv = dev(cuda, x0.copy())
            for _ in range(2):
                pmg.v_cycle(ctx, L - 1, xv, bd, use_graph=True)
            out[impl] = (xd.cpu().numpy(), xv.cpu().numpy())
    finally:
        pmg.set_smoother_impl("auto")
    assert np.array_equal(out["plane"][0], out["sweep"][0])
    assert np.array_equal(out["plane"][1], out["sweep"][1])


# Device GMRES with the V-cycle preconditioner (krylov.cpp:24-171) against the
# reference's GMRES on the same right-hand side: identical iteration counts,
# residual histories and solutions within the precision of the preconditioner
# (double: 1e-9 relative; mixed f32 V-cycle: 1e-4 on the history, whose
# entries are true f64 residual norms).
@pytest.mark.parametrize("mode", ["double", "mixed"])
@pytest.mark.parametrize("case", [(2, 2, 5), (3, 1, 4), (3, 3, 3), (3, 5, 2)], ids=lambda c: f"d{c[0]}k{c[1]}L{c[2]}")
def test_gmres_vs_reference(pmg, cuda, case, mode):
    dim, k, L = case
    ref64 = refbind.RefMg(dim, k, L, prec=0)
    ref32 = refbind.RefMg(dim, k, L, prec=1)
    b = refbind.compute_rhs(dim, k, L, 1)
    tol = 1e-10
    xr, itr, hr = refbind.gmres(ref64, ref32, mode == "mixed", b, tol, restart=10, max_iterations=50)
    op = pmg.make_multigrid_context(dim, k, L, dtype=np.float64)
    prec = op if mode == "double" else pmg.make_multigrid_context(dim, k, L, dtype=np.float32)
    xd = cuda.zeros(b.size, dtype=cuda.float64, device="cuda")
    st = pmg.gmres(op, prec, dev(cuda, b), xd, tol, restart=10, max_iterations=50)
    assert st.iterations == itr, (st.iterations, itr)
    h = np.asarray(st.residual_history)
    assert h.shape == hr.shape, (h, hr)
    htol = 1e-9 if mode == "double" else 1e-4
    assert np.allclose(h, hr, rtol=htol, atol=htol * hr[0]), (h, hr)
    assert rel(xd.cpu().numpy(), xr) < (1e-9 if mode == "double" else 1e-6)


# Device right-hand side and L2 error against the reference's compute_rhs and
# the host quadrature (operator.cpp:283-411): rhs relative 1e-14 (f64), L2
# error relative 1e-9 (both evaluate u_h - u pointwise at the same Gauss points).
@pytest.mark.parametrize("case", [(2, 1, 5), (2, 4, 4), (3, 1, 4), (3, 2, 4), (3, 5, 2), (3, 7, 2)],
                         ids=lambda c: f"d{c[0]}k{c[1]}L{c[2]}")
def test_device_rhs_and_l2(pmg, cuda, case):
    dim, k, L = case
    ctx = pmg.make_multigrid_context(dim, k, L, dtype=np.float64)
    lev = ctx.levels[-1]
    for f, kind in [("one", 0), ("sin", 1)]:
        want = refbind.compute_rhs(dim, k, L, kind)
        got = cuda.empty(want.size, dtype=cuda.float64, device="cuda")
        pmg.compute_rhs_device(lev, f, got)
        assert rel(got.cpu().numpy(), want) < 1e-14
    # a discrete solution-like field: the FMG-free sine interpolant plus noise
    x = np.random.default_rng(3).uniform(-1e-3, 1e-3, lev.level.total_dofs)
    e_host = pmg.l2_error(lev.level, x)
    e_dev = pmg.l2_error(lev, dev(cuda, x))
    e_ref = ctypes_double()
    assert refbind.lib().ref_l2_error_sin(dim, k, L, refbind.P(x), ctypes.byref(e_ref)) == 0
    assert abs(e_dev - e_host) <= 1e-9 * e_host, (e_dev, e_host)
    assert abs(e_dev - e_ref.value) <= 1e-9 * e_ref.value, (e_dev, e_ref.value)
    ctx32 = pmg.make_multigrid_context(dim, k, L, dtype=np.float32)
    got32 = cuda.empty(lev.level.total_dofs, dtype=cuda.float32, device="cuda")
    pmg.compute_rhs_device(ctx32.levels[-1], "sin", got32)
    assert rel(got32.cpu().numpy(), refbind.compute_rhs(dim, k, L, 1)) < 1e-6


# The size-dependent default: 3D k = 2 colours with >= 65536 patches run one
# thread per patch (vp_patch3d_kernel). One level large enough to select it,
# against the reference (multi-threaded CPU), f64 and f32, fused and boundary.
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_large_level_default_kernels(pmg, cuda, dtype):
    dim, k, L = 3, 2, 7
    ref = refbind.RefMg(dim, k, L, prec=0 if dtype == np.float64 else 1, threads=8)
    ctx = pmg.make_multigrid_context(dim, k, L, dtype=dtype)
    lev = ctx.levels[-1]
    x0, b = inputs(lev.level.total_dofs, dtype, seed=5)
    for variant in ["fused", "boundary"]:
        xd = dev(cuda, x0.copy())
        pmg.smooth(lev, xd, dev(cuda, b), variant)
        want = ref.smooth(L - 1, x0, b, variant)
        assert rel(xd.cpu().numpy(), want) < TOL[dtype], (variant, rel(xd.cpu().numpy(), want))


# restrict3d_kernel (the z-marching restriction) is selected for k = 1, 2, 4
# on fine levels of >= 96 nodes per direction; the cases above are smaller
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("case", [(3, 1, 7), (3, 2, 6), (3, 4, 5)], ids=lambda c: f"d{c[0]}k{c[1]}L{c[2]}")
def test_restrict3d_large(pmg, cuda, case, dtype):
    dim, k, L = case
    ref = refbind.RefMg(dim, k, L, prec=0 if dtype == np.float64 else 1)
    ctx = pmg.make_multigrid_context(dim, k, L, dtype=dtype)
    c, f = ctx.levels[-2], ctx.levels[-1]
    rf, _ = inputs(f.level.total_dofs, dtype, seed=9)
    rc = cuda.zeros(c.level.total_dofs, dtype=cuda.float64 if dtype == np.float64 else cuda.float32, device="cuda")
    pmg.restrict_vector(c, f, dev(cuda, rf), rc)
    assert rel(rc.cpu().numpy(), ref.restrict(L - 2, rf)) < TOL[dtype]
    if dtype == np.float64 and k == 2:
        x0, b = inputs(f.level.total_dofs, dtype)
        xd = dev(cuda, x0.copy())
        pmg.v_cycle(ctx, L - 1, xd, dev(cuda, b))
        assert rel(xd.cpu().numpy(), ref.vcycle(L - 1, x0, b)) < 1e-11


@pytest.mark.parametrize("case", [(2, 6), (4, 5), (1, 7), (3, 5)], ids=lambda c: f"k{c[0]}L{c[1]}")
def test_restrict_slab_ranges(pmg, cuda, case):
    """Owned-plane restriction (pmg_restrict_slab, the slab V-cycle's) on
    sub-ranges of coarse planes, from a local slab of the fine vector, equals
    the full restriction bitwise (restrict3d_kernel's node values do not
    depend on the z chunking)."""
    k, L = case
    ctx = pmg.make_multigrid_context(3, k, L)
    c, f = ctx.levels[-2], ctx.levels[-1]
    mf = f.level.dofs_per_dim
    mc = (mf - 1) // 2
    rf, _ = inputs(f.level.total_dofs, np.float64, seed=4)
    rfd = dev(cuda, rf)
    full = cuda.zeros(c.level.total_dofs, dtype=cuda.float64, device="cuda")
    pmg.restrict_vector(c, f, rfd, full)
    full = full.cpu().numpy().reshape(mc, mc * mc)
    for q0, q1 in ((0, mc), (0, 1), (3, 11), (mc // 2, mc), (mc - 1, mc), (k, 2 * k + 1)):
        # fine planes the range depends on, as a local slab
        c_lo = max(0, (q0 + 1) // k - (1 if (q0 + 1) % k == 0 else 0))
        pz0 = 2 * c_lo * k
        pz1 = min(2 * (q1 // k) * k + 2 * k, mf)
        local = rfd[pz0 * mf * mf:pz1 * mf * mf].clone()
        rc = cuda.zeros((q1 - q0) * mc * mc, dtype=cuda.float64, device="cuda")
        pmg.restrict_slab(c, f, local, pz0, rc, q0, q0, q1)
        assert np.array_equal(rc.cpu().numpy().reshape(q1 - q0, mc * mc), full[q0:q1]), (q0, q1)


# prolong2d_kernel / restrict2d_kernel on levels with many tiles
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("case", [(2, 1, 9), (2, 2, 8), (2, 3, 7), (2, 5, 6), (2, 7, 6)],
                         ids=lambda c: f"d{c[0]}k{c[1]}L{c[2]}")
def test_transfers2d_large(pmg, cuda, case, dtype):
    dim, k, L = case
    ref = refbind.RefMg(dim, k, L, prec=0 if dtype == np.float64 else 1)
    ctx = pmg.make_multigrid_context(dim, k, L, dtype=dtype)
    c, f = ctx.levels[-2], ctx.levels[-1]
    tdt = cuda.float64 if dtype == np.float64 else cuda.float32
    xc, _ = inputs(c.level.total_dofs, dtype, seed=7)
    rf, _ = inputs(f.level.total_dofs, dtype, seed=9)
    base = dev(cuda, rf.copy())
    pmg.prolongate(c, f, dev(cuda, xc), base, accumulate=True)
    assert rel(base.cpu().numpy(), rf.astype(np.float64) + ref.prolongate(L - 2, xc)) < TOL[dtype]
    rc = cuda.zeros(c.level.total_dofs, dtype=tdt, device="cuda")
    pmg.restrict_vector(c, f, dev(cuda, rf), rc)
    assert rel(rc.cpu().numpy(), ref.restrict(L - 2, rf)) < TOL[dtype]
