"""ctypes binding of the C-ABI (include/pmg_b200.h).

The shared library is built in-tree (paper_2405_19004_b200/libpmg_b200.so,
see __graft_entry__.build()). There is no fallback: if the library is missing
every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PMG_B200_LIB: an alternative in-tree build (A/B experiments of kernel variants)
LIB_PATH = os.environ.get("PMG_B200_LIB") or os.path.join(_HERE, "libpmg_b200.so")

PMG_OK, PMG_ERR_INVALID, PMG_ERR_RUNTIME, PMG_ERR_DIVERGENCE, PMG_ERR_CUDA = range(5)
PMG_F64, PMG_F32 = 0, 1
VARIANTS = {"global": 0, "separate": 1, "fused": 2, "boundary": 3, "naive": 100}

# (name, restype, argtypes) for every symbol declared in include/pmg_b200.h
_vp, _i, _i64, _d = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
_pi64, _pd, _pi = ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)
SIGNATURES = [
    ("pmg_last_error", ctypes.c_char_p, []),
    ("pmg_version", _i, []),
    ("pmg_device_info", _i, [_i, _pi, _pi, _pi, _pi]),
    ("pmg_level_create", _i, [_i, _i, _i, _i, _i, ctypes.POINTER(_vp)]),
    ("pmg_level_destroy", _i, [_vp]),
    ("pmg_level_info", _i, [_vp, _pi64, _pi64, _pi64]),
    ("pmg_smooth", _i, [_vp, _i, _vp, _vp, _vp]),
    ("pmg_smooth_host", _i, [_vp, _i, _vp, _vp]),
    ("pmg_smooth_color", _i, [_vp, _i, _i, _vp, _vp, _vp]),
    ("pmg_smooth_color_slab", _i, [_vp, _i, _i, _vp, _vp, _i64, _i64, _i, _i, _vp]),
    ("pmg_apply_laplacian", _i, [_vp, _vp, _vp, _vp]),
    ("pmg_apply_laplacian_host", _i, [_vp, _vp, _vp]),
    ("pmg_compute_residual", _i, [_vp, _vp, _vp, _vp, _vp]),
    ("pmg_compute_residual_host", _i, [_vp, _vp, _vp, _vp]),
    ("pmg_prolongate", _i, [_vp, _vp, _vp, _vp, _i, _vp]),
    ("pmg_prolongate_host", _i, [_vp, _vp, _vp, _vp]),
    ("pmg_restrict_vector", _i, [_vp, _vp, _vp, _vp, _vp]),
    ("pmg_restrict_vector_host", _i, [_vp, _vp, _vp, _vp]),
    ("pmg_vector_norm", _i, [_vp, _vp, _pd, _vp]),
    ("pmg_norm2", _i, [_vp, _i64, _i, _i, _pd, _vp]),
    ("pmg_mg_create", _i, [_i, _i, _i, _i, _i, _i, ctypes.POINTER(_vp)]),
    ("pmg_mg_destroy", _i, [_vp]),
    ("pmg_mg_num_levels", _i, [_vp]),
    ("pmg_mg_level", _vp, [_vp, _i]),
    ("pmg_mg_set_smoothing", _i, [_vp, _i, _i]),
    ("pmg_mg_set_variant", _i, [_vp, _i]),
    ("pmg_v_cycle", _i, [_vp, _i, _vp, _vp, _i, _vp]),
    ("pmg_v_cycle_host", _i, [_vp, _i, _vp, _vp]),
    ("pmg_full_multigrid", _i, [_vp, ctypes.POINTER(_vp), _vp, _d, _i, _pi, _pd, _i, _vp]),
    ("pmg_compute_rhs_host", _i, [_i, _i, _i, _i, _pd]),
    ("pmg_l2_error_sin_host", _i, [_i, _i, _i, _pd, _pd]),
    ("pmg_gmres", _i, [_vp, _vp, _vp, _vp, _d, _i, _i, _pi, _pd, _i, _vp]),
    ("pmg_level_setup_data", _i, [_vp, _pd, _pd, _pd, _pd, _pd, _pd, _pd]),
    ("pmg_host_level_setup", _i, [_i, _i, _i] + [_pd] * 9 + [_pi]),
    ("pmg_launch_count", _i64, []),
    ("pmg_set_smoother_impl", _i, [_i]),
    ("pmg_compute_rhs", _i, [_vp, _i, _vp, _vp]),
    ("pmg_compute_residual_slab", _i, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp]),
    ("pmg_restrict_slab", _i, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _vp]),
    ("pmg_prolongate_slab", _i, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _i, _vp]),
    ("pmg_l2_error_sin", _i, [_vp, _vp, _pd, _vp]),
    ("pmg_get_smoother_impl", _i, []),
    ("pmg_smoother_kernel", _i, [_vp, _i, _i, _pi]),
    ("pmg_full_multigrid_host", _i, [_vp, ctypes.POINTER(_vp), _pd, _d, _i, _pi, _pd, _i]),
    ("pmg_vector_norm_host", _i, [_vp, _i64, _i, _i, _pd]),
    ("pmg_gmres_host", _i, [_vp, _vp, _pd, _pd, _d, _i, _i, _pi, _pd, _i]),
    ("pmg_quadrature_rule", _i, [_i, _pd, _pd]),
    ("pmg_compute_rhs_q", _i, [_vp, _vp, _vp, _vp]),
    ("pmg_l2_error_q", _i, [_vp, _vp, _vp, _pd, _vp]),
    ("pmg_mg_create_kind", _i, [_i, _i, _i, _i, _i, _i, _i, ctypes.POINTER(_vp)]),
    ("pmg_point_gauss_seidel", _i, [_vp, _vp, _vp, _vp]),
    ("pmg_point_gauss_seidel_host", _i, [_vp, _pd, _pd]),
    ("pmg_assemble_sparse_host", _i, [_i, _i, _i, _pi64, ctypes.POINTER(ctypes.c_int32), _pd, _pi64]),
    ("pmg_dd_create", _i, [_i, _pi, _i, _i, _i, _i, _i, _i, _i, ctypes.POINTER(_vp)]),
    ("pmg_dd_nccl_id", _i, [_vp]),
    ("pmg_dd_create_rank", _i, [_i, _i, _i, _vp, _i, _i, _i, _i, _i, _i, ctypes.POINTER(_vp)]),
    ("pmg_dd_destroy", _i, [_vp]),
    ("pmg_dd_info", _i, [_vp, _pi, _pi, _pi]),
    ("pmg_dd_slab", _i, [_vp, _i, _i, ctypes.POINTER(_vp), _pi64, _pi64, _pi64, _pi64]),
    ("pmg_dd_stream", _i, [_vp, _i, ctypes.POINTER(_vp), _pi]),
    ("pmg_dd_scatter_host", _i, [_vp, _i, _vp]),
    ("pmg_dd_gather_host", _i, [_vp, _i, _vp]),
    ("pmg_dd_set_smoothing", _i, [_vp, _i, _i]),
    ("pmg_dd_smooth", _i, [_vp]),
    ("pmg_dd_set_graph", _i, [_vp, _i]),
    ("pmg_dd_v_cycle", _i, [_vp]),
    ("pmg_dd_residual_norm", _i, [_vp, _pd]),
    ("pmg_dd_full_multigrid", _i, [_vp, ctypes.POINTER(_vp), _d, _i, _pi, _pd, _i]),
    ("pmg_dd_synchronize", _i, [_vp]),
    ("pmg_dd_plan", _i64, [_i, _i, _i, _i, _i, _pi64, _i64]),
]

_lib = None


def load():
    """Load the in-tree C-ABI library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class DivergenceError(RuntimeError):
    """pmg::DivergenceError (multigrid.hpp:22-29): carries the residual history."""

    def __init__(self, msg, residual_history=None):
        super().__init__(msg)
        self.residual_history = list(residual_history or [])


def check(status: int, what: str = "", history=None) -> None:
    if status == PMG_OK:
        return
    msg = load().pmg_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == PMG_ERR_INVALID:
        raise ValueError(text)
    if status == PMG_ERR_DIVERGENCE:
        raise DivergenceError(text, history)
    raise RuntimeError(text)
