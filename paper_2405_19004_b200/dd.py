"""Slab domain decomposition of the colourised vertex-patch smoother.

SURVEY.md §8e: patches of one colour are independent, so the smoother shards
along the slowest direction (z) by vertex planes; only the colour-to-colour
dependency crosses ranks. Rank g owns the vertex planes v_z in [a_g, b_g].

  * It reads dof planes [k(a-1)-1, k(b+1)-1] and writes [k(a-1), k(b+1)-2]
    (closure / interior of its patches, patches.cpp:71,114), so it keeps that
    range of global planes locally ("lo".."hi").
  * After colour c only ONE side of an interface writes near it: the patch at
    v = b_g (if its parity is the colour's z-bit) updates planes
    [k b_g - 1, k b_g + k - 2] that rank g+1 reads, else the patch at
    v = b_g + 1 = a_{g+1} updates [k b_g, k b_g + k - 1] that rank g reads.
    So per colour and interface one one-directional message of k planes.
  * The boundary-layer patches (v in {a, b}) run first, the message is posted,
    the interior patches run while it is in flight, and the next colour waits
    for it (overlap of the halo exchange with interior patches).

The colour order and the per-patch arithmetic are unchanged, so the P-rank
result equals the 1-rank result bitwise on the GPU.

The driver is generic over the colour kernel (the CUDA slab kernel on the
GPU; the numpy oracle in the CPU tests) and over the transport
(torch.distributed NCCL / gloo, or device copies between virtual ranks).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class SlabPlan:
    world: int
    rank: int
    k: int
    n: int  # cells per direction along x, y
    nz: int  # cells along z of the global box (n: unit cube; world*n: stacked box)
    a: int  # first owned vertex plane (1-based lattice vertex index)
    b: int  # last owned vertex plane
    lo: int  # first global dof plane held locally
    hi: int  # last global dof plane held locally (inclusive)
    own_lo: int  # dof planes this rank is the owner of (for gathers), inclusive
    own_hi: int

    @property
    def m(self) -> int:
        return self.n * self.k - 1

    @property
    def mz(self) -> int:
        return self.nz * self.k - 1

    @property
    def nplanes(self) -> int:
        return self.hi - self.lo + 1

    @property
    def plane_size(self) -> int:
        return self.m * self.m


def make_plan(world: int, rank: int, k: int, level: int, stack: int = 1) -> SlabPlan:
    """Split the nz-1 interior vertex planes of a box of 2^level cells along
    x, y and stack * 2^level along z (stack = 1: the reference's unit cube;
    stack = world: weak scaling with one cube per rank) into `world`
    contiguous ranges."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    n = 1 << level
    nz = stack * n
    nv = nz - 1
    if nv < world:
        raise ValueError(f"{nv} vertex planes cannot be split over {world} ranks")
    a = 1 + (rank * nv) // world
    b = ((rank + 1) * nv) // world
    mz = nz * k - 1
    lo = max(0, k * (a - 1) - 1)
    hi = min(mz - 1, k * (b + 1) - 1)
    own_lo = 0 if rank == 0 else k * (a - 1)
    own_hi = mz - 1 if rank == world - 1 else k * b - 1
    return SlabPlan(world, rank, k, n, nz, a, b, lo, hi, own_lo, own_hi)


def colour_nonempty(n: int, color: int) -> bool:
    """x / y patch counts of the colour are non-zero (patches.cpp:24-33)."""
    for a in range(2):
        cnt = n // 2 if (color >> a) & 1 else n // 2 - 1
        if cnt <= 0:
            return False
    return True


@dataclass(frozen=True)
class ColourStep:
    early: list  # vertex ranges (lo, hi) to smooth before the message is posted
    late: list  # vertex ranges smoothed while the message is in flight
    sends: list  # (peer, first global plane, nplanes)
    recvs: list  # (peer, first global plane, nplanes)


def colour_step(p: SlabPlan, color: int) -> ColourStep:
    if not colour_nonempty(p.n, color):
        return ColourStep([], [], [], [])
    zb = (color >> 2) & 1
    k = p.k
    sends, recvs, early = [], [], set()
    if p.rank + 1 < p.world:  # upper interface, with rank+1
        if p.b % 2 == zb:
            sends.append((p.rank + 1, k * p.b - 1, k))
            early.add(p.b)
        else:
            recvs.append((p.rank + 1, k * p.b, k))
    if p.rank > 0:  # lower interface, with rank-1 (whose b is a-1)
        bl = p.a - 1
        if bl % 2 == zb:
            recvs.append((p.rank - 1, k * bl - 1, k))
        else:
            sends.append((p.rank - 1, k * bl, k))
            early.add(p.a)
    early = sorted(early)
    lo_v = p.a + (1 if p.a in early else 0)
    hi_v = p.b - (1 if (p.b in early and p.b != p.a) else 0)
    late = [(lo_v, hi_v)] if lo_v <= hi_v else []
    return ColourStep([(v, v) for v in early], late, sends, recvs)


class SlabSmoother:
    """One colourised multiplicative smoothing step on this rank's slab.

    kernel(color, vz_lo, vz_hi): smooth the colour's patches of this slab
    whose vertex z lies in [vz_lo, vz_hi] (in place on the local x).
    comm: object with post(sends, recvs) -> handle, handle.wait(); sends /
    recvs carry (peer, first local plane, nplanes).
    """

    def __init__(self, plan: SlabPlan, kernel, comm):
        self.plan, self.kernel, self.comm = plan, kernel, comm
        self.steps = [colour_step(plan, c) for c in range(8)]

    def smooth(self):
        p = self.plan
        for c in range(8):
            st = self.steps[c]
            for lo, hi in st.early:
                self.kernel(c, lo, hi)
            h = None
            if st.sends or st.recvs:
                h = self.comm.post([(q, g0 - p.lo, n) for q, g0, n in st.sends],
                                   [(q, g0 - p.lo, n) for q, g0, n in st.recvs])
            for lo, hi in st.late:
                self.kernel(c, lo, hi)
            if h is not None:
                h.wait()


class TorchDistComm:
    """Plane messages through torch.distributed point-to-point (NCCL on the
    GPU box, gloo in the CPU tests). `x` is the local flat vector."""

    def __init__(self, x, plane_size: int):
        self.x, self.ps = x, plane_size

    def post(self, sends, recvs):
        import torch.distributed as dist

        ops = []
        for q, l0, n in sends:
            ops.append(dist.P2POp(dist.isend, self.x[l0 * self.ps:(l0 + n) * self.ps], q))
        for q, l0, n in recvs:
            ops.append(dist.P2POp(dist.irecv, self.x[l0 * self.ps:(l0 + n) * self.ps], q))
        reqs = dist.batch_isend_irecv(ops)

        class H:
            def wait(self_inner):
                for r in reqs:
                    r.wait()

        return H()


def virtual_smooth(plans, kernels, xs):
    """P slabs in ONE process (one device): colour by colour, all ranks'
    early patches, then the plane copies, then the late patches. Used to test
    the decomposition on a single GPU (and on the CPU with the oracle)."""
    steps = [[colour_step(p, c) for c in range(8)] for p in plans]
    for c in range(8):
        for r, p in enumerate(plans):
            for lo, hi in steps[r][c].early:
                kernels[r](c, lo, hi)
        for r, p in enumerate(plans):
            for q, g0, n in steps[r][c].sends:
                src = xs[r][(g0 - p.lo) * p.plane_size:(g0 - p.lo + n) * p.plane_size]
                dst_p = plans[q]
                xs[q][(g0 - dst_p.lo) * p.plane_size:(g0 - dst_p.lo + n) * p.plane_size] = src
        for r, p in enumerate(plans):
            for lo, hi in steps[r][c].late:
                kernels[r](c, lo, hi)


def scatter_global(plan: SlabPlan, x_global):
    """Local slab (planes lo..hi) of a global flat vector."""
    return x_global[plan.lo * plan.plane_size:(plan.hi + 1) * plan.plane_size]


def owned_part(plan: SlabPlan, x_local):
    """The planes this rank owns, out of its local slab."""
    a = (plan.own_lo - plan.lo) * plan.plane_size
    b = (plan.own_hi + 1 - plan.lo) * plan.plane_size
    return x_local[a:b]


def gpu_kernel(level_ctx, plan: SlabPlan, x_local, b_local, variant="fused"):
    """The CUDA colour kernel of this slab (pmg_smooth_color_slab)."""
    from .pmg import smooth_color_slab

    def run(color, vz_lo, vz_hi):
        smooth_color_slab(level_ctx, color, x_local, b_local, plan.lo, plan.nz, vz_lo, vz_hi, variant)

    return run


class StagedComm:
    """Host-staged plane messages over a CPU backend (gloo). Only for
    exercising the multi-rank driver when several ranks share one GPU (NCCL
    refuses two ranks per device); the product path is TorchDistComm/NCCL."""

    def __init__(self, x, plane_size: int):
        self.x, self.ps = x, plane_size

    def post(self, sends, recvs):
        import torch.distributed as dist

        ops, bufs = [], []
        for q, l0, n in sends:
            ops.append(dist.P2POp(dist.isend, self.x[l0 * self.ps:(l0 + n) * self.ps].cpu(), q))
        for q, l0, n in recvs:
            buf = self.x.new_empty(n * self.ps, device="cpu")
            bufs.append((l0, n, buf))
            ops.append(dist.P2POp(dist.irecv, buf, q))
        reqs = dist.batch_isend_irecv(ops) if ops else []
        x, ps = self.x, self.ps

        class H:
            def wait(self_inner):
                for r in reqs:
                    r.wait()
                for l0, n, buf in bufs:
                    x[l0 * ps:(l0 + n) * ps].copy_(buf)

        return H()
