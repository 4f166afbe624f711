"""The coarse V-cycle operator: on the largest level with at
most PMG_COARSE_MAT_N (default 3375) unknowns the parent's coarse correction
is one GEMV with the precomputed V-cycle matrix of that level. These cases
pass through it (3D k=1 L5 and k=2 L5: 15^3 = 3375-unknown level; k=4 L3:
the 15^3 level too; 2D k=2 L6: 31^2), against the reference's recursive
V-cycle (multigrid.cpp:313-348) with changed smoothing counts and variants,
which must rebuild the operator (MultigridContext::pre_smooth / post_smooth /
variant, multigrid.hpp:37-40). f64 1e-12 relative; f32 by the residual
criterion (1e-5 of ||b||).
"""

import os

import numpy as np
import pytest

import refbind

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1
CASES = [(3, 1, 5), (3, 2, 5), (3, 4, 3), (2, 2, 6)]
SETTINGS = [(1, 1, "fused"), (2, 1, "boundary"), (1, 2, "separate"), (1, 1, "fused")]


def rel(a, b):
    nb = np.linalg.norm(np.asarray(b, np.float64))
    return np.linalg.norm(np.asarray(a, np.float64) - np.asarray(b, np.float64)) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def pmg(cuda):
    import paper_2405_19004_b200 as p

    if not refbind.available():
        pytest.fail("oracle/_ref/libpmg_ref.so missing: run __graft_entry__.build() where /root/reference exists")
    return p


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"d{c[0]}k{c[1]}L{c[2]}")
def test_vcycle_through_coarse_operator(pmg, cuda, case, dtype):
    dim, k, L = case
    f64 = dtype == np.float64
    ref = refbind.RefMg(dim, k, L, prec=0 if f64 else 1, threads=THREADS)
    ref64 = ref if f64 else refbind.RefMg(dim, k, L, prec=0, threads=THREADS)
    ctx = pmg.make_multigrid_context(dim, k, L, dtype=dtype)
    n = ctx.levels[-1].level.total_dofs
    # the hierarchy does contain a level the operator is built for
    assert any(lv.level.total_dofs <= 3375 for lv in ctx.levels[1:-1])
    x0, b = refbind.fill_uniform(5, n, n)
    x0, b = x0.astype(dtype), b.astype(dtype)
    b64 = b.astype(np.float64)
    for pre, post, variant in SETTINGS:
        ctx.pre_smooth, ctx.post_smooth, ctx.variant = pre, post, variant
        ref.set_smoothing(pre, post)
        ref.set_variant(variant)
        want = ref.vcycle(L - 1, x0, b)
        for use_graph in (False, True):
            xd = cuda.from_numpy(x0.copy()).cuda()
            pmg.v_cycle(ctx, L - 1, xd, cuda.from_numpy(b).cuda(), use_graph=use_graph)
            got = xd.cpu().numpy()
            if f64:
                assert rel(got, want) < 1e-12, (pre, post, variant, use_graph, rel(got, want))
            else:
                r_got = ref64.residual(L - 1, got.astype(np.float64), b64)
                r_want = ref64.residual(L - 1, want.astype(np.float64), b64)
                err = np.linalg.norm(r_got - r_want) / np.linalg.norm(b64)
                assert err < 1e-5, (pre, post, variant, use_graph, err)


def test_coarse_gemv_is_deterministic(pmg, cuda):
    """Two contexts (two operators built independently) give bitwise equal
    V-cycles: the column sweep and the GEMV's reduction order are fixed."""
    out = []
    for _ in range(2):
        ctx = pmg.make_multigrid_context(3, 2, 5)
        n = ctx.levels[-1].level.total_dofs
        x0, b = refbind.fill_uniform(9, n, n)
        xd = cuda.from_numpy(x0.copy()).cuda()
        for _ in range(2):
            pmg.v_cycle(ctx, 4, xd, cuda.from_numpy(b).cuda(), use_graph=True)
        out.append(xd.cpu().numpy())
    assert np.array_equal(out[0], out[1])
