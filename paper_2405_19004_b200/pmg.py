"""Python host mirror of the reference `pmg` interface, over the C-ABI.

Same names, argument meaning and error behaviour as /root/reference/proj/
include/pmg/*.hpp (the parity tests read like the SPEC's examples):

  build_hierarchy / dof_index / CartesianLevel     mesh.hpp:16-35
  make_level_context / LevelContext                level_context.hpp:17-29
  make_multigrid_context / MultigridContext        multigrid.hpp:34-54
  smooth                                           smoother.hpp:45-47
  apply_laplacian / compute_rhs / l2_error         operator.hpp:47-64
  prolongate / restrict_vector                     multigrid.hpp:56-63
  v_cycle / full_multigrid / FmgStats              multigrid.hpp:68-86
  vector_norm / compute_residual                   multigrid.hpp:89-92
  gmres / SolveStats (+ mixed precision)           krylov.hpp:16-39
  DivergenceError                                  multigrid.hpp:22-29

Vectors are either torch CUDA tensors (device path: the C-ABI enqueues on the
current torch stream, x is updated in place) or numpy arrays (host path: the
*_host C-ABI entry points copy in, compute on the GPU, copy out). Every
computation runs in the CUDA library; nothing here does arithmetic on the
vectors.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import PMG_F32, PMG_F64, VARIANTS, DivergenceError, check

__all__ = [
    "CartesianLevel", "build_hierarchy", "dof_index", "LevelContext", "make_level_context",
    "MultigridContext", "make_multigrid_context", "SmootherVariant", "smooth", "smooth_color", "smooth_color_slab",
    "apply_laplacian", "compute_residual", "prolongate", "restrict_vector", "v_cycle",
    "full_multigrid", "FmgStats", "vector_norm", "compute_rhs", "l2_error", "gmres", "SolveStats",
    "DivergenceError", "set_smoother_impl", "get_smoother_impl", "compute_rhs_device",
    "compute_residual_slab", "restrict_slab", "prolongate_slab", "smoother_kernel", "KERNEL_NAMES",
    "MultiGpuContext", "nccl_unique_id", "quadrature_points", "point_gauss_seidel", "assemble_sparse", "SMOOTHER_KINDS",
]

_SMOOTHER_IMPLS = {"auto": 0, "line": 1, "plane": 2, "sweep": 3, "patch": 4}


def set_smoother_impl(impl: str = "auto") -> None:
    """Select the smoother kernel organisation for later calls (A/B
    measurement; no reference counterpart): "auto" (per-degree default),
    "line" (line-per-thread kernel everywhere), "plane" (plane-streaming
    kernel, 3D fused/boundary, degree <= 2, one launch per colour) or "sweep"
    (the plane kernel with all colours of a step in one persistent launch)."""
    if impl not in _SMOOTHER_IMPLS:
        raise ValueError(f"smoother impl must be one of {sorted(_SMOOTHER_IMPLS)}")
    check(_lib.load().pmg_set_smoother_impl(_SMOOTHER_IMPLS[impl]), "set_smoother_impl")


def get_smoother_impl() -> str:
    code = _lib.load().pmg_get_smoother_impl()
    return {v: k for k, v in _SMOOTHER_IMPLS.items()}[code]


KERNEL_NAMES = {0: "vp_smooth_kernel", 1: "vp_point_kernel", 2: "vp_patch2d_kernel", 3: "vp_patch3d_kernel",
                4: "vp_smooth_plane_kernel", 5: "vp_smooth_pp_kernel", 6: "naive_smooth_kernel"}


def smoother_kernel(ctx, variant="fused", color: int = 0) -> str:
    """Name of the kernel a colour launch of smooth() runs on this level under
    the current set_smoother_impl choice (pmg_smoother_kernel)."""
    out = ctypes.c_int(-1)
    check(_lib.load().pmg_smoother_kernel(ctx.handle, _variant_code(variant), int(color), ctypes.byref(out)),
          "smoother_kernel")
    return KERNEL_NAMES[out.value]


class SmootherVariant:
    """smoother.hpp:21-27 (+ the straightforward global-memory comparator)."""

    global_ = "global"
    separate = "separate"
    fused = "fused"
    boundary = "boundary"
    naive = "naive"


# ---------------------------------------------------------------------------
# mesh (mesh.hpp)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class CartesianLevel:
    level: int = 1
    dim: int = 2
    degree: int = 1

    @property
    def cells_per_dim(self) -> int:
        return 1 << self.level

    @property
    def dofs_per_dim(self) -> int:
        return self.cells_per_dim * self.degree - 1

    @property
    def spacing(self) -> float:
        return 1.0 / self.cells_per_dim

    @property
    def total_dofs(self) -> int:
        return self.dofs_per_dim ** self.dim


def build_hierarchy(dim: int, degree: int, finest_level: int) -> list[CartesianLevel]:
    if dim not in (2, 3):
        raise ValueError(f"build_hierarchy: dim must be 2 or 3, got {dim}")
    if degree < 1:
        raise ValueError("build_hierarchy: degree must be >= 1")
    if finest_level < 1:
        raise ValueError("build_hierarchy: finest_level must be >= 1")
    return [CartesianLevel(l, dim, degree) for l in range(1, finest_level + 1)]


def dof_index(level: CartesianLevel, multi_index) -> int:
    if len(multi_index) != level.dim:
        raise ValueError("dof_index: multi-index size does not match dim")
    m = level.dofs_per_dim
    idx, stride = 0, 1
    for a, v in enumerate(multi_index):
        if not 0 <= v < m:
            raise IndexError(f"dof_index: component {a} out of range")
        idx += v * stride
        stride *= m
    return idx


# ---------------------------------------------------------------------------
# array plumbing
# ---------------------------------------------------------------------------


def _dtype_code(dtype) -> int:
    dt = np.dtype(dtype)
    if dt == np.float64:
        return PMG_F64
    if dt == np.float32:
        return PMG_F32
    raise ValueError(f"unsupported dtype {dtype} (float32 / float64 only)")


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


class _Arr:
    """Classifies an argument as a device (torch CUDA) or host (numpy) array."""

    def __init__(self, a, n: int, dtype_code: int, name: str, writable: bool):
        if _is_torch(a):
            import torch

            if not a.is_cuda:
                raise ValueError(f"{name}: torch tensors must live on a CUDA device")
            want = torch.float64 if dtype_code == PMG_F64 else torch.float32
            if a.dtype != want:
                raise ValueError(f"{name}: dtype {a.dtype} does not match the context ({want})")
            if not a.is_contiguous():
                raise ValueError(f"{name}: tensor must be contiguous")
            if a.numel() != n:
                raise ValueError(f"{name}: vector size does not match level")
            self.device = True
            self.ptr = ctypes.c_void_p(a.data_ptr())
            self.obj = a
        else:
            if not isinstance(a, np.ndarray):
                raise TypeError(f"{name}: expected a numpy array or a torch CUDA tensor")
            want = np.float64 if dtype_code == PMG_F64 else np.float32
            if a.dtype != want:
                raise ValueError(f"{name}: dtype {a.dtype} does not match the context ({np.dtype(want)})")
            if a.size != n:
                raise ValueError(f"{name}: vector size does not match level")
            if not a.flags.c_contiguous or (writable and not a.flags.writeable):
                raise ValueError(f"{name}: array must be C-contiguous (and writable)")
            self.device = False
            self.ptr = ctypes.c_void_p(a.ctypes.data)
            self.obj = a


def _stream(arrs, ctx=None) -> ctypes.c_void_p:
    """torch's current stream ON THE DEVICE of the vectors; every device vector
    must live on one device, and on the context's device when one is given
    (the C-ABI dereferences them on that device)."""
    import torch

    devs = set()
    for a in arrs:
        t = a.obj if isinstance(a, _Arr) else a
        if _is_torch(t) and t.is_cuda:
            devs.add(t.device.index if t.device.index is not None else torch.cuda.current_device())
    if len(devs) > 1:
        raise ValueError(f"vectors on different CUDA devices {sorted(devs)}")
    want = getattr(ctx, "device", None) if ctx is not None else None
    if want is not None and devs and devs != {want}:
        raise ValueError(f"vectors on cuda:{devs.pop()} but the context lives on cuda:{want}")
    dev = devs.pop() if devs else (want if want is not None else torch.cuda.current_device())
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _same_kind(*arrs):
    kinds = {a.device for a in arrs}
    if len(kinds) != 1:
        raise ValueError("mix of host (numpy) and device (torch) vectors")
    return kinds.pop()


# ---------------------------------------------------------------------------
# level context
# ---------------------------------------------------------------------------


class LevelContext:
    """Per-level immutable setup (level_context.hpp:17-26), resident on the GPU."""

    def __init__(self, handle, level: CartesianLevel, dtype, device: int, owner=None):
        self._h = ctypes.c_void_p(handle)
        self.level = level
        self.dtype = np.dtype(dtype)
        self.device = device
        self._owner = owner  # keeps a MultigridContext alive for borrowed levels

    @property
    def handle(self):
        return self._h

    @property
    def _code(self):
        return _dtype_code(self.dtype)

    def setup_data(self) -> dict:
        """The f64 setup uploaded for this level (for parity tests)."""
        k, d = self.level.degree, self.level.dim
        ni, nc = 2 * k - 1, 2 * k + 1
        out = {
            "S": np.zeros((ni, ni)), "lambda": np.zeros(ni), "mass_if": np.zeros((ni, nc)),
            "stiff_if": np.zeros((ni, nc)), "prolongation": np.zeros((nc, k + 1)),
            "cell_mass": np.zeros((k + 1, k + 1)), "cell_stiffness": np.zeros((k + 1, k + 1)),
        }
        P = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
        check(_lib.load().pmg_level_setup_data(
            self._h, P(out["S"]), P(out["lambda"]), P(out["mass_if"]), P(out["stiff_if"]),
            P(out["prolongation"]), P(out["cell_mass"]), P(out["cell_stiffness"])), "setup_data")
        return out

    def __del__(self):
        if self._owner is None and getattr(self, "_h", None) and _lib._lib is not None:
            _lib._lib.pmg_level_destroy(self._h)
            self._h = None


def make_level_context(level: CartesianLevel, dtype=np.float64, device: int = 0) -> LevelContext:
    lib = _lib.load()
    h = ctypes.c_void_p()
    check(lib.pmg_level_create(level.dim, level.degree, level.level, _dtype_code(dtype), device,
                               ctypes.byref(h)), "make_level_context")
    return LevelContext(h.value, level, dtype, device)


# ---------------------------------------------------------------------------
# smoother / operator / transfers
# ---------------------------------------------------------------------------


def _variant_code(variant) -> int:
    if isinstance(variant, int):
        return variant
    try:
        return VARIANTS[variant]
    except KeyError:
        raise ValueError(f"unknown smoother variant {variant!r}") from None


def smooth(ctx: LevelContext, x, b, variant="fused", threads: int = 1, ws=None) -> None:
    """One colourised multiplicative vertex-patch step, x updated in place
    (smoother.hpp:45-47). `threads`/`ws` are accepted for signature parity;
    the GPU grid replaces parallel_for."""
    n = ctx.level.total_dofs
    xa = _Arr(x, n, ctx._code, "x", True)
    ba = _Arr(b, n, ctx._code, "b", False)
    v = _variant_code(variant)
    lib = _lib.load()
    if _same_kind(xa, ba):
        check(lib.pmg_smooth(ctx.handle, v, xa.ptr, ba.ptr, _stream((xa, ba), ctx)), "smooth")
    else:
        check(lib.pmg_smooth_host(ctx.handle, v, xa.ptr, ba.ptr), "smooth")


def smooth_color(ctx: LevelContext, color: int, x, b, variant="fused") -> None:
    """One colour of a smoothing step (device vectors only)."""
    n = ctx.level.total_dofs
    xa = _Arr(x, n, ctx._code, "x", True)
    ba = _Arr(b, n, ctx._code, "b", False)
    if not (xa.device and ba.device):
        raise ValueError("smooth_color: device (torch CUDA) vectors only")
    check(_lib.load().pmg_smooth_color(ctx.handle, _variant_code(variant), color, xa.ptr, ba.ptr,
                                       _stream((xa, ba), ctx)), "smooth_color")


def smooth_color_slab(ctx: LevelContext, color: int, x_local, b_local, z_offset: int, nz_cells: int,
                      vz_lo: int, vz_hi: int, variant="fused") -> None:
    """One colour on a z-slab of a (possibly stacked) 3D box (device vectors
    holding the global dof planes z >= z_offset); see dd.py."""
    lev = ctx.level
    plane = lev.dofs_per_dim ** 2
    for name, v in (("x_local", x_local), ("b_local", b_local)):
        if not _is_torch(v) or not v.is_cuda or v.numel() % plane:
            raise ValueError(f"{name}: device vector of whole dof planes required")
    xa = _Arr(x_local, x_local.numel(), ctx._code, "x_local", True)
    ba = _Arr(b_local, b_local.numel(), ctx._code, "b_local", False)
    check(_lib.load().pmg_smooth_color_slab(ctx.handle, _variant_code(variant), color, xa.ptr, ba.ptr,
                                            int(z_offset), int(nz_cells), int(vz_lo), int(vz_hi),
                                            _stream((xa,), ctx)), "smooth_color_slab")


def apply_laplacian(ctx: LevelContext, x, y, mode: str = "colored", threads: int = 1) -> None:
    """y = A_l x (operator.hpp:47-50)."""
    n = ctx.level.total_dofs
    xa = _Arr(x, n, ctx._code, "x", False)
    ya = _Arr(y, n, ctx._code, "y", True)
    lib = _lib.load()
    if _same_kind(xa, ya):
        check(lib.pmg_apply_laplacian(ctx.handle, xa.ptr, ya.ptr, _stream((xa, ya), ctx)), "apply_laplacian")
    else:
        check(lib.pmg_apply_laplacian_host(ctx.handle, xa.ptr, ya.ptr), "apply_laplacian")


def compute_residual(ctx: LevelContext, x, b, r, threads: int = 1) -> None:
    """r = b - A x (multigrid.hpp:90-92)."""
    n = ctx.level.total_dofs
    xa = _Arr(x, n, ctx._code, "x", False)
    ba = _Arr(b, n, ctx._code, "b", False)
    ra = _Arr(r, n, ctx._code, "r", True)
    lib = _lib.load()
    if _same_kind(xa, ba, ra):
        check(lib.pmg_compute_residual(ctx.handle, xa.ptr, ba.ptr, ra.ptr, _stream((xa, ba, ra), ctx)), "compute_residual")
    else:
        check(lib.pmg_compute_residual_host(ctx.handle, xa.ptr, ba.ptr, ra.ptr), "compute_residual")


def _check_pair(coarse: LevelContext, fine: LevelContext, what: str):
    cl, fl = coarse.level, fine.level
    if fl.level != cl.level + 1 or fl.degree != cl.degree or fl.dim != cl.dim:
        raise ValueError(f"{what}: levels are not consecutive")


def prolongate(coarse: LevelContext, fine: LevelContext, x_coarse, x_fine, accumulate: bool = False) -> None:
    """x_fine = P x_coarse (multigrid.hpp:56-58); accumulate gives +=."""
    _check_pair(coarse, fine, "prolongate")
    xc = _Arr(x_coarse, coarse.level.total_dofs, fine._code, "x_coarse", False)
    xf = _Arr(x_fine, fine.level.total_dofs, fine._code, "x_fine", True)
    lib = _lib.load()
    if _same_kind(xc, xf):
        check(lib.pmg_prolongate(coarse.handle, fine.handle, xc.ptr, xf.ptr, int(accumulate),
                                 _stream((xc, xf), fine)), "prolongate")
    else:
        if accumulate:
            raise ValueError("prolongate: accumulate needs device vectors")
        check(lib.pmg_prolongate_host(coarse.handle, fine.handle, xc.ptr, xf.ptr), "prolongate")


def restrict_vector(coarse: LevelContext, fine: LevelContext, r_fine, r_coarse) -> None:
    """r_coarse = P^T r_fine (multigrid.hpp:61-63)."""
    _check_pair(coarse, fine, "restrict_vector")
    rf = _Arr(r_fine, fine.level.total_dofs, fine._code, "r_fine", False)
    rc = _Arr(r_coarse, coarse.level.total_dofs, fine._code, "r_coarse", True)
    lib = _lib.load()
    if _same_kind(rf, rc):
        check(lib.pmg_restrict_vector(coarse.handle, fine.handle, rf.ptr, rc.ptr, _stream((rf, rc), fine)),
              "restrict_vector")
    else:
        check(lib.pmg_restrict_vector_host(coarse.handle, fine.handle, rf.ptr, rc.ptr), "restrict_vector")


# ---------------------------------------------------------------------------
# slab operations of the z-slab domain decomposition (dd.py). Arrays are CUDA
# tensors holding the global dof planes [zoff, zoff + numel / m^2).
# ---------------------------------------------------------------------------


def _slab(ctx: LevelContext, a, name: str, writable: bool):
    m = ctx.level.dofs_per_dim
    if not (_is_torch(a) and a.is_cuda):
        raise TypeError(f"{name}: slab operations take CUDA tensors")
    if a.numel() % (m * m):
        raise ValueError(f"{name}: not a whole number of planes")
    return _Arr(a, a.numel(), ctx._code, name, writable), a.numel() // (m * m)


def compute_residual_slab(ctx: LevelContext, x, b, r, zoff: int, p0: int, p1: int) -> None:
    """r = b - A x on global planes [p0, p1) (multigrid.cpp:268-276); x, b, r
    hold the same planes [zoff, zoff + n)."""
    ax, n = _slab(ctx, x, "x", False)
    ab, nb = _slab(ctx, b, "b", False)
    ar, nr = _slab(ctx, r, "r", True)
    if not n == nb == nr:
        raise ValueError("compute_residual_slab: x, b, r must hold the same planes")
    check(_lib.load().pmg_compute_residual_slab(ctx.handle, ax.ptr, ab.ptr, ar.ptr, zoff, n, p0, p1,
                                                _stream([x, b, r], ctx)),
          "compute_residual_slab")


def restrict_slab(coarse: LevelContext, fine: LevelContext, rf, zoff_f: int, rc, zoff_c: int, q0: int,
                  q1: int) -> None:
    """Coarse planes [q0, q1) of R r_f (multigrid.cpp:162-248)."""
    af, nf = _slab(fine, rf, "rf", False)
    ac, nc = _slab(coarse, rc, "rc", True)
    check(_lib.load().pmg_restrict_slab(coarse.handle, fine.handle, af.ptr, zoff_f, nf, ac.ptr, zoff_c, nc, q0, q1,
                                        _stream([rf, rc], fine)), "restrict_slab")


def prolongate_slab(coarse: LevelContext, fine: LevelContext, xc, zoff_c: int, xf, zoff_f: int, f0: int, f1: int,
                    accumulate: bool = True) -> None:
    """Fine planes [f0, f1) (+)= P x_c (multigrid.cpp:71-160)."""
    ac, nc = _slab(coarse, xc, "xc", False)
    af, nf = _slab(fine, xf, "xf", True)
    check(_lib.load().pmg_prolongate_slab(coarse.handle, fine.handle, ac.ptr, zoff_c, nc, af.ptr, zoff_f, nf, f0, f1,
                                          1 if accumulate else 0, _stream([xc, xf], fine)), "prolongate_slab")


def vector_norm(v, device: int = 0) -> float:
    """Euclidean norm (multigrid.cpp:260-266), deterministic device reduction."""
    lib = _lib.load()
    out = ctypes.c_double()
    if _is_torch(v):
        code = _dtype_code(str(v.dtype).replace("torch.", ""))
        a = _Arr(v, v.numel(), code, "v", False)
        check(lib.pmg_norm2(a.ptr, v.numel(), code, v.device.index or 0, ctypes.byref(out),
                            _stream((a,))), "vector_norm")
        return out.value
    import torch  # host vector: stage through the device like every other op

    t = torch.from_numpy(np.ascontiguousarray(v)).to(f"cuda:{device}")
    return vector_norm(t)


# ---------------------------------------------------------------------------
# multigrid context / V-cycle / FMG
# ---------------------------------------------------------------------------


class MultigridContext:
    """Level hierarchy + device workspaces (multigrid.hpp:34-49). Index 0 is
    mesh level 1 (one interior vertex)."""

    def __init__(self, handle, dim, degree, finest_level, variant, dtype, device):
        self._h = ctypes.c_void_p(handle)
        self.dtype = np.dtype(dtype)
        self.device = device
        self._variant = variant
        self._pre, self._post = 1, 1
        lib = _lib.load()
        self.levels = [
            LevelContext(lib.pmg_mg_level(self._h, li), lev, dtype, device, owner=self)
            for li, lev in enumerate(build_hierarchy(dim, degree, finest_level))
        ]

    @property
    def handle(self):
        return self._h

    @property
    def variant(self):
        return self._variant

    @variant.setter
    def variant(self, v):
        check(_lib.load().pmg_mg_set_variant(self._h, _variant_code(v)), "variant")
        self._variant = v

    @property
    def pre_smooth(self):
        return self._pre

    @pre_smooth.setter
    def pre_smooth(self, n):
        check(_lib.load().pmg_mg_set_smoothing(self._h, int(n), self._post), "pre_smooth")
        self._pre = int(n)

    @property
    def post_smooth(self):
        return self._post

    @post_smooth.setter
    def post_smooth(self, n):
        check(_lib.load().pmg_mg_set_smoothing(self._h, self._pre, int(n)), "post_smooth")
        self._post = int(n)

    def __del__(self):
        if getattr(self, "_h", None) and _lib._lib is not None:
            _lib._lib.pmg_mg_destroy(self._h)
            self._h = None


SMOOTHER_KINDS = {"vertex_patch": 0, "point_gs": 1}  # SmootherKind, multigrid.hpp:16-20


def make_multigrid_context(dim: int, degree: int, finest_level: int, variant="fused",
                           kind: str = "vertex_patch", threads: int = 1, dtype=np.float64,
                           device: int = 0) -> MultigridContext:
    """multigrid.hpp:51-54. kind "point_gs" smooths with one lexicographic
    point Gauss-Seidel sweep per pre/post step (f64 only, like the reference;
    ValueError otherwise; RuntimeError past the reference's 1e7-nonzero CSR
    budget)."""
    if kind not in SMOOTHER_KINDS:
        raise ValueError(f"kind must be one of {sorted(SMOOTHER_KINDS)}")
    build_hierarchy(dim, degree, finest_level)  # same argument validation
    lib = _lib.load()
    h = ctypes.c_void_p()
    check(lib.pmg_mg_create_kind(dim, degree, finest_level, _dtype_code(dtype), _variant_code(variant),
                                 SMOOTHER_KINDS[kind], device, ctypes.byref(h)), "make_multigrid_context")
    ctx = MultigridContext(h.value, dim, degree, finest_level, variant, dtype, device)
    ctx.kind = kind
    return ctx


def point_gauss_seidel(ctx: LevelContext, x, b) -> None:
    """One forward lexicographic Gauss-Seidel sweep on the level's operator
    (point_gauss_seidel(assemble_sparse(level), x, b), smoother.cpp:160-166),
    f64, x in place."""
    if ctx.dtype != np.float64:
        raise ValueError("point Gauss-Seidel runs in f64 only")
    n = ctx.level.total_dofs
    xa = _Arr(x, n, PMG_F64, "x", True)
    ba = _Arr(b, n, PMG_F64, "b", False)
    lib = _lib.load()
    if _same_kind(xa, ba):
        check(lib.pmg_point_gauss_seidel(ctx.handle, xa.ptr, ba.ptr, _stream((xa, ba), ctx)), "point_gauss_seidel")
    else:
        check(lib.pmg_point_gauss_seidel_host(ctx.handle, ctypes.cast(xa.ptr, ctypes.POINTER(ctypes.c_double)),
                                              ctypes.cast(ba.ptr, ctypes.POINTER(ctypes.c_double))),
              "point_gauss_seidel")


def assemble_sparse(level: CartesianLevel):
    """CSR matrix of the level operator (operator.cpp:194-281), host:
    (row_ptr int64[N+1], cols int32[nnz], vals float64[nnz])."""
    lib = _lib.load()
    nnz = ctypes.c_int64()
    check(lib.pmg_assemble_sparse_host(level.dim, level.degree, level.level, None, None, None, ctypes.byref(nnz)),
          "assemble_sparse")
    rp = np.zeros(level.total_dofs + 1, dtype=np.int64)
    cols = np.zeros(nnz.value, dtype=np.int32)
    vals = np.zeros(nnz.value)
    check(lib.pmg_assemble_sparse_host(level.dim, level.degree, level.level,
                                       rp.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                       cols.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                       vals.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(nnz)),
          "assemble_sparse")
    return rp, cols, vals


def v_cycle(ctx: MultigridContext, li: int, x, b, use_graph: bool = False) -> None:
    """One V-cycle on level index li (multigrid.hpp:68-69), x in place."""
    if not 0 <= li < len(ctx.levels):
        raise ValueError("v_cycle: level index out of range")
    lev = ctx.levels[li]
    n = lev.level.total_dofs
    xa = _Arr(x, n, lev._code, "x", True)
    ba = _Arr(b, n, lev._code, "b", False)
    lib = _lib.load()
    if _same_kind(xa, ba):
        check(lib.pmg_v_cycle(ctx.handle, li, xa.ptr, ba.ptr, int(use_graph), _stream((xa, ba), ctx.levels[-1])),
              "v_cycle")
    else:
        check(lib.pmg_v_cycle_host(ctx.handle, li, xa.ptr, ba.ptr), "v_cycle")


@dataclass
class FmgStats:
    """multigrid.hpp:74-78."""

    iterations: int = 0
    residual_history: list = field(default_factory=list)


def full_multigrid(ctx: MultigridContext, rhs_per_level, x, tol: float, max_iterations: int = 100) -> FmgStats:
    """Alg. 2 (multigrid.hpp:80-86): nested iteration then V-cycles until
    ||b - A x|| <= tol ||b||. f64 contexts only. Raises DivergenceError."""
    import torch

    if ctx.dtype != np.float64:
        raise ValueError("full_multigrid: f64 contexts only")
    if tol <= 0:
        raise ValueError("full_multigrid: tol must be positive")
    L = len(ctx.levels)
    if len(rhs_per_level) != L:
        raise ValueError("full_multigrid: need one rhs per level")
    dev = f"cuda:{ctx.device}"
    rhs_dev = [r if _is_torch(r) else torch.from_numpy(np.ascontiguousarray(r, dtype=np.float64)).to(dev)
               for r in rhs_per_level]
    for r, lev in zip(rhs_dev, ctx.levels):
        _Arr(r, lev.level.total_dofs, PMG_F64, "rhs", False)
    host_x = not _is_torch(x)
    xd = torch.zeros(ctx.levels[-1].level.total_dofs, dtype=torch.float64, device=dev) if host_x else x
    _Arr(xd, ctx.levels[-1].level.total_dofs, PMG_F64, "x", True)
    ptrs = (ctypes.c_void_p * L)(*[r.data_ptr() for r in rhs_dev])
    cap = max_iterations + 2
    hist = np.full(cap, np.nan)
    its = ctypes.c_int(0)
    st = _lib.load().pmg_full_multigrid(
        ctx.handle, ptrs, ctypes.c_void_p(xd.data_ptr()), float(tol), int(max_iterations), ctypes.byref(its),
        hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), cap,
        ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    history = [float(h) for h in hist[: its.value + 1]]
    check(st, "full_multigrid", history)
    if host_x:
        np.copyto(x, xd.cpu().numpy())
    return FmgStats(its.value, history)


def quadrature_points(level: CartesianLevel, device: int = 0):
    """The reference's quadrature points of a level (operator.cpp:283-411:
    (k+2)-point Gauss per direction and cell) as a float64 CUDA tensor of shape
    (cells * (k+2)^d, d): cells lexicographic, direction 0 fastest, then the
    points of a cell, direction 0 fastest (the fq layout of pmg_compute_rhs_q)."""
    import torch

    k, d, n = level.degree, level.dim, level.cells_per_dim
    pts = np.zeros(k + 2)
    wts = np.zeros(k + 2)
    check(_lib.load().pmg_quadrature_rule(k, pts.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                          wts.ctypes.data_as(ctypes.POINTER(ctypes.c_double))), "quadrature_rule")
    dev = f"cuda:{device}"
    xi = torch.from_numpy(pts).to(dev)
    c = torch.arange(n, dtype=torch.float64, device=dev)
    h = 1.0 / n
    # axis a of the (cell_{d-1}, ..., cell_0, q_{d-1}, ..., q_0) grid
    cells = torch.meshgrid(*([c] * d), indexing="ij")          # (c_{d-1}.., c_0) order below
    qs = torch.meshgrid(*([xi] * d), indexing="ij")
    coords = []
    for a in range(d):
        ca = cells[d - 1 - a].reshape(-1, 1)                     # cell coordinate of direction a
        qa = qs[d - 1 - a].reshape(1, -1)
        coords.append(((ca + qa) * h).reshape(-1))
    return torch.stack(coords, dim=1)


def _field_values(level: CartesianLevel, f, device: int):
    """f at the level's quadrature points: f(pts) with pts a (P, d) float64
    CUDA tensor -> P values (the torch form of ScalarField, operator.hpp:41)."""
    import torch

    pts = quadrature_points(level, device)
    v = f(pts)
    v = torch.as_tensor(v, dtype=torch.float64, device=pts.device).reshape(-1).contiguous()
    if v.numel() != pts.shape[0]:
        raise ValueError("field must return one value per quadrature point")
    return v


_KINDS = {"one": 0, "sin": 1}


def compute_rhs(level: CartesianLevel, f="one") -> np.ndarray:
    """b_i = int f phi_i (operator.hpp:58-59) as a host f64 array: f = 'one'
    (f = 1), 'sin' (d pi^2 prod sin(pi x_a)), or any field f(pts) -> values
    evaluated on the device at the reference's quadrature points and assembled
    there (pmg_compute_rhs_q)."""
    if callable(f):
        import torch

        ctx = make_level_context(level, np.float64, 0)
        out = torch.zeros(level.total_dofs, dtype=torch.float64, device="cuda:0")
        compute_rhs_device(ctx, f, out)
        return out.cpu().numpy()
    if f not in _KINDS:
        raise ValueError("compute_rhs: f must be 'one', 'sin' or a callable field")
    out = np.zeros(level.total_dofs)
    check(_lib.load().pmg_compute_rhs_host(level.dim, level.degree, level.level, _KINDS[f],
                                           out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))), "compute_rhs")
    return out


def compute_rhs_device(ctx: LevelContext, f, out) -> None:
    """compute_rhs on the device into `out` (a CUDA tensor of the level's
    dtype). 'one' / 'sin': the tensor power of the 1D load vector, exact on
    the uniform level; a callable field: its values at the quadrature points,
    integrated cell by cell against the basis (operator.cpp:283-344)."""
    a = _Arr(out, ctx.level.total_dofs, ctx._code, "b", True)
    if callable(f):
        fq = _field_values(ctx.level, f, ctx.device)
        check(_lib.load().pmg_compute_rhs_q(ctx.handle, ctypes.c_void_p(fq.data_ptr()), a.ptr,
                                            _stream([out], ctx)), "compute_rhs")
        return
    if f not in _KINDS:
        raise ValueError("compute_rhs: f must be 'one', 'sin' or a callable field")
    check(_lib.load().pmg_compute_rhs(ctx.handle, _KINDS[f], a.ptr, _stream([out], ctx)), "compute_rhs")


def l2_error(level, x, u_exact="sin") -> float:
    """L2 error ||u_h - u|| (operator.hpp:62-64) with the (k+2)^d-point Gauss
    rule, u = prod sin(pi x_a) ('sin') or any field u(pts) -> values. With a
    LevelContext and a CUDA tensor it runs on the device."""
    if callable(u_exact):
        import torch

        if isinstance(level, LevelContext):
            ctx = level
        else:
            ctx = make_level_context(level, np.float64, 0)
        xd = x if (_is_torch(x) and x.is_cuda) else torch.from_numpy(
            np.ascontiguousarray(x, dtype=ctx.dtype)).to(f"cuda:{ctx.device}")
        a = _Arr(xd, ctx.level.total_dofs, ctx._code, "x", False)
        uq = _field_values(ctx.level, u_exact, ctx.device)
        out = ctypes.c_double()
        check(_lib.load().pmg_l2_error_q(ctx.handle, a.ptr, ctypes.c_void_p(uq.data_ptr()), ctypes.byref(out),
                                         _stream([xd], ctx)), "l2_error")
        return out.value
    if u_exact != "sin":
        raise ValueError("l2_error: u_exact must be 'sin' or a callable field")
    if isinstance(level, LevelContext) and _is_torch(x) and x.is_cuda:
        a = _Arr(x, level.level.total_dofs, level._code, "x", False)
        out = ctypes.c_double()
        check(_lib.load().pmg_l2_error_sin(level.handle, a.ptr, ctypes.byref(out), _stream([x], level)), "l2_error")
        return out.value
    if isinstance(level, LevelContext):
        level = level.level
    xh = x.detach().cpu().numpy() if _is_torch(x) else np.ascontiguousarray(x, dtype=np.float64)
    xh = np.ascontiguousarray(xh, dtype=np.float64)
    if xh.size != level.total_dofs:
        raise ValueError("l2_error: vector size does not match level")
    out = ctypes.c_double()
    check(_lib.load().pmg_l2_error_sin_host(level.dim, level.degree, level.level,
                                            xh.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                            ctypes.byref(out)), "l2_error")
    return out.value


# ---------------------------------------------------------------------------
# Krylov (krylov.hpp)
# ---------------------------------------------------------------------------


@dataclass
class SolveStats:
    iterations: int = 0
    residual_history: list = field(default_factory=list)
    l2_error: float | None = None
    wall_seconds: float = 0.0


def gmres(op_ctx: MultigridContext, prec_ctx: MultigridContext, b, x, tol: float, restart: int = 30,
          max_iterations: int = 200) -> SolveStats:
    """Right-preconditioned GMRES(restart) in f64 with one V-cycle of
    `prec_ctx` as preconditioner: an f32 context is the paper's mixed
    precision mode (krylov.cpp:152-171), an f64 context the double mode."""
    import time

    import torch

    n = op_ctx.levels[-1].level.total_dofs
    dev = f"cuda:{op_ctx.device}"
    bd = b if _is_torch(b) else torch.from_numpy(np.ascontiguousarray(b, dtype=np.float64)).to(dev)
    host_x = not _is_torch(x)
    xd = torch.zeros(n, dtype=torch.float64, device=dev) if host_x else x
    _Arr(bd, n, PMG_F64, "b", False)
    _Arr(xd, n, PMG_F64, "x", True)
    cap = max_iterations + 8
    hist = np.full(cap, np.nan)
    its = ctypes.c_int(0)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    st = _lib.load().pmg_gmres(op_ctx.handle, prec_ctx.handle, ctypes.c_void_p(bd.data_ptr()),
                               ctypes.c_void_p(xd.data_ptr()), float(tol), int(restart), int(max_iterations),
                               ctypes.byref(its), hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), cap,
                               ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - t0
    h = [float(v) for v in hist if not np.isnan(v)]
    if -1.0 in h:
        h = h[: h.index(-1.0)]
    check(st, "gmres", h)
    if host_x:
        np.copyto(x, xd.cpu().numpy())
    return SolveStats(its.value, h, None, wall)


# ---------------------------------------------------------------------------
# Multi-GPU (the C-ABI's slab domain decomposition, pmg_dd_*; csrc/dd.cu)
# ---------------------------------------------------------------------------
DD_TRANSPORTS = {"copy": 0, "nccl": 1}


class MultiGpuContext:
    """make_multigrid_context + smooth / v_cycle / full_multigrid
    (multigrid.hpp:51-86) on a z-slab decomposition over several devices,
    driven by the C++ host code of the library (one process).

    devices: one device id per rank (repeats allowed with transport "copy":
    virtual ranks sharing a GPU). The handle owns x and b of the finest
    level; `scatter` / `gather` move global host vectors in and out.
    Results equal the single-device ones bitwise (norms to rounding)."""

    def __init__(self, devices, dim: int, degree: int, finest_level: int, stack: int = 1,
                 dtype=np.float64, variant="fused", transport: str = "copy", _handle=None):
        lib = _lib.load()
        self.dim, self.degree, self.finest_level, self.stack = dim, degree, finest_level, stack
        self.dtype = np.dtype(dtype)
        m = (1 << finest_level) * degree - 1
        self.mz = stack * (1 << finest_level) * degree - 1
        self.total_dofs = m * m * self.mz
        self._devices = list(devices) if devices is not None else None
        if _handle is not None:
            self._h = _handle
        else:
            if transport not in DD_TRANSPORTS:
                raise ValueError(f"transport must be one of {sorted(DD_TRANSPORTS)}")
            devs = (ctypes.c_int * len(devices))(*devices)
            h = ctypes.c_void_p()
            check(lib.pmg_dd_create(len(devices), devs, dim, degree, finest_level, stack, _dtype_code(dtype),
                                    _variant_code(variant), DD_TRANSPORTS[transport], ctypes.byref(h)),
                  "MultiGpuContext")
            self._h = h
        w, lr, nd = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        check(lib.pmg_dd_info(self._h, ctypes.byref(w), ctypes.byref(lr), ctypes.byref(nd)), "dd_info")
        self.world, self.local_ranks, self.decomposed_levels = w.value, lr.value, nd.value

    @classmethod
    def for_rank(cls, world: int, rank: int, device: int, nccl_id: bytes, dim: int, degree: int,
                 finest_level: int, stack: int = 1, dtype=np.float64, variant="fused"):
        """One process per GPU over NCCL (nccl_id from `nccl_unique_id()` on
        rank 0, shared by the caller, e.g. torch.distributed)."""
        lib = _lib.load()
        buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        h = ctypes.c_void_p()
        check(lib.pmg_dd_create_rank(world, rank, device, buf, dim, degree, finest_level, stack,
                                     _dtype_code(dtype), _variant_code(variant), ctypes.byref(h)),
              "MultiGpuContext.for_rank")
        return cls([device], dim, degree, finest_level, stack, dtype, variant, _handle=h)

    def slab(self, local: int = 0, which: str = "x"):
        """(device pointer, first global plane, planes, own_lo, own_hi)."""
        p = ctypes.c_void_p()
        z0, np_, lo, hi = (ctypes.c_int64() for _ in range(4))
        check(_lib.load().pmg_dd_slab(self._h, local, 0 if which == "x" else 1, ctypes.byref(p), ctypes.byref(z0),
                                      ctypes.byref(np_), ctypes.byref(lo), ctypes.byref(hi)), "dd_slab")
        return p.value, z0.value, np_.value, lo.value, hi.value

    def slab_tensor(self, local: int = 0, which: str = "x"):
        """The slab of local rank `local` as a torch CUDA tensor (no copy; the
        memory stays owned by the context)."""
        import torch

        ptr, _, nplanes, _, _ = self.slab(local, which)
        m = (1 << self.finest_level) * self.degree - 1
        n = nplanes * m * m
        _, rank = self.stream(local)
        dev = self._devices[local] if self._devices else torch.cuda.current_device()

        class _View:
            __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8" if self.dtype == np.float64 else "<f4",
                                        "data": (ptr, False), "version": 3, "strides": None}

        with torch.cuda.device(dev):
            return torch.as_tensor(_View(), device=f"cuda:{dev}")

    def stream(self, local: int = 0):
        """(cudaStream_t of local rank `local`, its global rank)."""
        s, r = ctypes.c_void_p(), ctypes.c_int()
        check(_lib.load().pmg_dd_stream(self._h, local, ctypes.byref(s), ctypes.byref(r)), "dd_stream")
        return s.value, r.value

    def _host(self, a, writable):
        if not isinstance(a, np.ndarray) or a.dtype != self.dtype or a.size != self.total_dofs \
                or not a.flags.c_contiguous or (writable and not a.flags.writeable):
            raise ValueError(f"expected a contiguous {self.dtype} host array of {self.total_dofs} values")
        return ctypes.c_void_p(a.ctypes.data)

    def scatter(self, which: str, global_host: np.ndarray) -> None:
        check(_lib.load().pmg_dd_scatter_host(self._h, 0 if which == "x" else 1, self._host(global_host, False)),
              "dd_scatter")

    def gather(self, which: str = "x", out: np.ndarray | None = None) -> np.ndarray:
        out = np.zeros(self.total_dofs, dtype=self.dtype) if out is None else out
        check(_lib.load().pmg_dd_gather_host(self._h, 0 if which == "x" else 1, self._host(out, True)), "dd_gather")
        return out

    def set_smoothing(self, pre: int, post: int) -> None:
        check(_lib.load().pmg_dd_set_smoothing(self._h, pre, post), "dd_set_smoothing")

    def smooth(self) -> None:
        check(_lib.load().pmg_dd_smooth(self._h), "dd_smooth")

    def set_graph(self, enable: bool = True) -> None:
        """Replay the smoothing step as one captured CUDA graph (local ranks on
        one device)."""
        check(_lib.load().pmg_dd_set_graph(self._h, int(enable)), "dd_set_graph")

    def v_cycle(self) -> None:
        check(_lib.load().pmg_dd_v_cycle(self._h), "dd_v_cycle")

    def residual_norm(self) -> float:
        out = ctypes.c_double()
        check(_lib.load().pmg_dd_residual_norm(self._h, ctypes.byref(out)), "dd_residual_norm")
        return out.value

    def full_multigrid(self, rhs_per_level, tol: float, max_iterations: int = 100) -> FmgStats:
        """Alg. 2 on the decomposition (f64); the solution stays in x
        (`gather("x")`). rhs_per_level: global host arrays, one per level."""
        L = self.finest_level
        if len(rhs_per_level) != L:
            raise ValueError("full_multigrid: need one rhs per level")
        arrs = [np.ascontiguousarray(r, dtype=np.float64) for r in rhs_per_level]
        ptrs = (ctypes.c_void_p * L)(*[a.ctypes.data for a in arrs])
        cap = max_iterations + 2
        hist = np.full(cap, np.nan)
        its = ctypes.c_int(0)
        st = _lib.load().pmg_dd_full_multigrid(self._h, ptrs, float(tol), int(max_iterations), ctypes.byref(its),
                                              hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), cap)
        history = [float(h) for h in hist[: its.value + 1]]
        check(st, "full_multigrid", history)
        return FmgStats(its.value, history)

    def synchronize(self) -> None:
        check(_lib.load().pmg_dd_synchronize(self._h), "dd_synchronize")

    def __del__(self):
        if getattr(self, "_h", None) and _lib._lib is not None:
            _lib._lib.pmg_dd_destroy(self._h)
            self._h = None


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the library (rank 0 of MultiGpuContext.for_rank)."""
    buf = ctypes.create_string_buffer(128)
    check(_lib.load().pmg_dd_nccl_id(buf), "nccl_unique_id")
    return buf.raw
