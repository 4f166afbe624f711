"""GPU: compute_rhs / l2_error with a general (non-separable) field
(operator.hpp:55-64): the field evaluated on the device at the reference's
quadrature points, assembled / integrated there (pmg_compute_rhs_q,
pmg_l2_error_q), against the reference's own compute_rhs / l2_error with the
same field (oracle/ref_capi.cpp f_gen)."""

import ctypes

import numpy as np
import pytest

import refbind

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not refbind.available(), reason="oracle/_ref not built")]


def f_gen(p):
    import torch

    z = p[:, 2] if p.shape[1] > 2 else torch.full_like(p[:, 0], 0.25)
    return torch.exp(p[:, 0] - 0.5 * p[:, 1]) * (1.0 + p[:, 1] ** 2) * torch.cos(2.0 * p[:, 0] * z + p[:, 1])


@pytest.mark.parametrize("dim,k,L", [(2, 1, 4), (2, 3, 3), (2, 7, 2), (3, 1, 3), (3, 2, 3), (3, 4, 2), (3, 7, 1)])
def test_general_rhs_and_l2_vs_reference(cuda, dim, k, L):
    import paper_2405_19004_b200 as pmg

    lev = pmg.build_hierarchy(dim, k, L)[-1]
    b = pmg.compute_rhs(lev, f_gen)
    br = np.zeros(lev.total_dofs)
    assert refbind.lib().ref_compute_rhs(dim, k, L, 2, br.ctypes.data) == 0
    np.testing.assert_allclose(b, br, rtol=1e-12, atol=1e-14 * np.abs(br).max())
    # f32 context: same integrals rounded to f32
    ctx32 = pmg.make_level_context(lev, np.float32)
    b32 = cuda.zeros(lev.total_dofs, dtype=cuda.float32, device="cuda")
    pmg.compute_rhs_device(ctx32, f_gen, b32)
    np.testing.assert_allclose(b32.cpu().numpy(), br, rtol=1e-6, atol=1e-7 * np.abs(br).max())
    # l2 error of an arbitrary iterate against the same field
    x = np.random.default_rng(3).uniform(-1, 1, lev.total_dofs)
    e = pmg.l2_error(lev, x, f_gen)
    er = ctypes.c_double()
    assert refbind.lib().ref_l2_error_gen(dim, k, L, x.ctypes.data, ctypes.byref(er)) == 0
    assert abs(e - er.value) <= 1e-12 * er.value


def test_string_kinds_unchanged_through_general_path(cuda):
    """'sin' through the general path equals the tensor-power path."""
    import math

    import paper_2405_19004_b200 as pmg

    lev = pmg.build_hierarchy(3, 3, 3)[-1]
    b1 = pmg.compute_rhs(lev, "sin")

    def fsin(p):
        import torch

        return 3 * math.pi ** 2 * torch.prod(torch.sin(math.pi * p), dim=1)

    b2 = pmg.compute_rhs(lev, fsin)
    np.testing.assert_allclose(b2, b1, rtol=1e-12, atol=1e-14 * np.abs(b1).max())
