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

import numpy as np


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

    def __init__(self, plan: SlabPlan, kernel, comm, side_stream=None):
        self.plan, self.kernel, self.comm = plan, kernel, comm
        self.steps = [colour_step(plan, c) for c in range(8)]
        # optional torch.cuda.Stream: the boundary-layer patches and the plane
        # messages run on it, concurrently with the interior patches on the
        # current stream (they are independent patches of the same colour)
        self.side = side_stream

    def smooth(self):
        p = self.plan
        if self.side is not None:
            import torch
        for c in range(8):
            st = self.steps[c]
            sends = [(q, g0 - p.lo, n) for q, g0, n in st.sends]
            recvs = [(q, g0 - p.lo, n) for q, g0, n in st.recvs]
            h = None
            if self.side is None:
                for lo, hi in st.early:
                    self.kernel(c, lo, hi)
                if sends or recvs:
                    h = self.comm.post(sends, recvs)
                for lo, hi in st.late:
                    self.kernel(c, lo, hi)
                if h is not None:
                    h.wait()
                continue
            main = torch.cuda.current_stream()
            self.side.wait_stream(main)
            with torch.cuda.stream(self.side):
                for lo, hi in st.early:
                    self.kernel(c, lo, hi)
                if sends or recvs:
                    h = self.comm.post(sends, recvs)
                    h.wait()
            for lo, hi in st.late:
                self.kernel(c, lo, hi)
            main.wait_stream(self.side)


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


# ---------------------------------------------------------------------------
# SURVEY.md §8e "alternative to evaluate": ONE exchange per smoothing step
# instead of one per colour, bought with redundant halo patches. A patch at
# vertex v reads the dof planes of vertices v-1..v+1 and writes strictly
# between them. A rank owning vertex planes [a, b] (dof planes k(a-1) ..
# kb-1, the lowest of which is also written by vertex a-1) must therefore run
# the last colour on vertices [a-1, b], colour 6 on [a-2, b+1], ..., colour c
# on [a-1-(7-c), b+(7-c)]: the values each colour reads are then exact —
# received from their owner at the start of the step or recomputed from exact
# inputs by the owner's arithmetic — and the owned planes end equal to the
# single-domain step bitwise. The local slab holds the dof planes of
# vertices a-9 .. b+8; every non-owned plane of it arrives in one message
# per neighbour. Cost: the same bytes as the 8 per-colour messages, in one;
# sum_c (15 - 2c) = 64 extra colour vertex-planes of patches per rank.
DEEP = 8  # 2^d colours (3D)


def deep_halo_plan(plan: SlabPlan) -> SlabPlan:
    """`plan` with its local slab widened to the dof planes of vertices
    a - 9 .. b + 8 (clipped to the box); ownership unchanged."""
    k = plan.k
    lo = max(0, k * (plan.a - DEEP - 1) - 1)
    hi = min(plan.mz - 1, k * (plan.b + DEEP) - 1)
    return SlabPlan(plan.world, plan.rank, plan.k, plan.n, plan.nz, plan.a, plan.b, lo, hi, plan.own_lo,
                    plan.own_hi)


def deep_halo_messages(plans):
    """Per rank: (sends, recvs) of (peer, first global plane, nplanes) so every
    rank receives the non-owned planes of its widened slab from their owners."""
    msgs = [([], []) for _ in plans]
    for r, p in enumerate(plans):
        for q, o in enumerate(plans):
            if q == r:
                continue
            g0, g1 = max(p.lo, o.own_lo), min(p.hi, o.own_hi)
            if g0 <= g1:
                msgs[q][0].append((r, g0, g1 - g0 + 1))
                msgs[r][1].append((q, g0, g1 - g0 + 1))
    return msgs


def deep_colour_range(p: SlabPlan, color: int):
    """Vertex planes colour `color` smooths on this rank in the deep-halo step."""
    nv = p.nz - 1
    lo, hi = max(1, p.a - 1 - (DEEP - 1 - color)), min(nv, p.b + (DEEP - 1 - color))
    return (lo, hi) if lo <= hi and colour_nonempty(p.n, color) else None


class DeepHaloSmoother:
    """One smoothing step with a single halo exchange (see above). plan: a
    deep_halo_plan; sends / recvs: this rank's entry of deep_halo_messages;
    kernel(color, vz_lo, vz_hi) and comm as for SlabSmoother."""

    def __init__(self, plan: SlabPlan, sends, recvs, kernel, comm):
        self.plan, self.kernel, self.comm = plan, kernel, comm
        self.sends = [(q, g0 - plan.lo, n) for q, g0, n in sends]
        self.recvs = [(q, g0 - plan.lo, n) for q, g0, n in recvs]

    def smooth(self):
        if self.sends or self.recvs:
            self.comm.post(self.sends, self.recvs).wait()
        for c in range(8):
            r = deep_colour_range(self.plan, c)
            if r is not None:
                self.kernel(c, r[0], r[1])


def virtual_deep_smooth(plans, kernels, xs):
    """deep-halo step for P slabs in one process: owners' planes copied into
    every widened slab, then each rank's colours."""
    msgs = deep_halo_messages(plans)
    for r, p in enumerate(plans):
        for q, g0, n in msgs[r][1]:
            o = plans[q]
            xs[r][(g0 - p.lo) * p.plane_size:(g0 - p.lo + n) * p.plane_size] = \
                xs[q][(g0 - o.lo) * o.plane_size:(g0 - o.lo + n) * o.plane_size]
    for r, p in enumerate(plans):
        for c in range(8):
            rg = deep_colour_range(p, c)
            if rg is not None:
                kernels[r](c, rg[0], rg[1])


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


# ---------------------------------------------------------------------------
# The V-cycle on z-slabs (SURVEY.md §8e "rest of the V-cycle").
#
# Levels whose slabs are thick enough (every rank owns >= 2 H dof planes,
# H = 4k + 4) are decomposed; below that the level is agglomerated: its
# right-hand side is all-gathered and every rank runs the remaining V-cycle
# redundantly on the whole (small) level, so no broadcast is needed. On a
# decomposed level each rank keeps its vectors on the planes E = [lo - H,
# hi + H] (clipped), the smoother's slab [lo, hi] plus halo:
#
#   pre-smooth (SlabSmoother, per-colour one-directional plane messages)
#   halo(x)                      neighbours' owned planes -> E
#   r = b - A x on owned planes  (residual_slab), halo(r)
#   b_c = R r on coarse owned planes (restrict_slab), halo(b_c), x_c = 0
#   recurse; halo(x_c)
#   x += P x_c on [lo, hi]       (prolongate_slab; the halo planes of [lo, hi]
#                                 get the same update as their owner's copy)
#   post-smooth
#
# Every value is computed by the same per-output arithmetic as the
# single-domain V-cycle (multigrid.cpp:313-348), so P ranks reproduce it
# bitwise. The operations are supplied by a backend (GPU C-ABI slab entry
# points, or the numpy oracle in the CPU tests); messages by a communicator
# factory (torch.distributed NCCL / gloo).
# ---------------------------------------------------------------------------


def halo_width(k: int) -> int:
    return 4 * k + 4


@dataclass(frozen=True)
class LevelSlab:
    level: int
    plan: SlabPlan
    e0: int  # first global dof plane held (extended slab E)
    e1: int  # last (inclusive)

    @property
    def n(self) -> int:
        return self.e1 - self.e0 + 1


def level_slab(world: int, rank: int, k: int, level: int) -> LevelSlab:
    p = make_plan(world, rank, k, level)
    H = halo_width(k)
    return LevelSlab(level, p, max(0, p.lo - H), min(p.mz - 1, p.hi + H))


def decomposed_levels(world: int, k: int, finest: int) -> list:
    """Levels (finest first) on which every rank owns >= 2 H planes."""
    out = []
    for lev in range(finest, 1, -1):
        n = 1 << lev
        if n - 1 < world:
            break
        plans = [make_plan(world, r, k, lev) for r in range(world)]
        if min(p.own_hi - p.own_lo + 1 for p in plans) < 2 * halo_width(k):
            break
        out.append(lev)
    return out


def _exchange_specs(world: int, rank: int, slabs_by_rank):
    """(sends, recvs) of local-plane ranges that bring every plane of my E
    outside my owned range from its owner, and give my neighbours theirs."""
    me = slabs_by_rank[rank]
    sends, recvs = [], []
    for q in (rank - 1, rank + 1):
        if not 0 <= q < world:
            continue
        nb = slabs_by_rank[q]
        # planes of my E owned by q
        lo = max(me.e0, nb.plan.own_lo)
        hi = min(me.e1, nb.plan.own_hi)
        if lo <= hi:
            recvs.append((q, lo - me.e0, hi - lo + 1))
        # planes of q's E owned by me
        lo = max(nb.e0, me.plan.own_lo)
        hi = min(nb.e1, me.plan.own_hi)
        if lo <= hi:
            sends.append((q, lo - me.e0, hi - lo + 1))
    return sends, recvs


class SlabVCycle:
    """One V-cycle (pre = post = 1) of the slab-decomposed hierarchy.

    ops: backend with
      kernel(level, slab, x_view, b_view) -> colour kernel for SlabSmoother
      residual(level, x, b, r, e0, p0, p1)
      restrict(level_f, rf, e0_f, rc, e0_c, q0, q1)
      prolongate(level_f, xc, e0_c, xf, e0_f, f0, f1)        (accumulating)
      vcycle_full(level, b_full) -> x_full                    (agglomerated)
      zeros(n), view(a, start, count), owned_slice(...)
    comm(array, plane_size) -> object with post(sends, recvs).wait()
    allgather(array) -> list of arrays from all ranks (rank order)
    """

    def __init__(self, world, rank, k, finest, ops, comm, allgather):
        self.world, self.rank, self.k, self.finest = world, rank, k, finest
        self.ops, self.comm, self.allgather = ops, comm, allgather
        self.dd_levels = decomposed_levels(world, k, finest)
        if not self.dd_levels or self.dd_levels[0] != finest:
            raise ValueError("finest level too thin for the slab decomposition on this many ranks")
        self.agg = self.dd_levels[-1] - 1  # first agglomerated level
        self.slabs = {lev: [level_slab(world, r, k, lev) for r in range(world)] for lev in self.dd_levels}
        self.ex = {lev: _exchange_specs(world, rank, self.slabs[lev]) for lev in self.dd_levels}
        self.ps = {lev: ((1 << lev) * k - 1) ** 2 for lev in range(1, finest + 1)}
        # work vectors per decomposed level (finest: x, b are the caller's)
        self.r, self.bc, self.xc = {}, {}, {}
        for lev in self.dd_levels:
            n = self.slabs[lev][rank].n * self.ps[lev]
            self.r[lev] = ops.zeros(n)
            if lev - 1 in self.slabs:
                nc = self.slabs[lev - 1][rank].n * self.ps[lev - 1]
            else:
                nc = self.ps[lev - 1] * ((1 << (lev - 1)) * k - 1)  # the whole agglomerated level
            self.bc[lev] = ops.zeros(nc)
            self.xc[lev] = ops.zeros(nc)

    def slab(self, lev) -> LevelSlab:
        return self.slabs[lev][self.rank]

    def halo(self, lev, a):
        sends, recvs = self.ex[lev]
        if sends or recvs:
            self.comm(a, self.ps[lev]).post(sends, recvs).wait()

    def _smooth(self, lev, x, b):
        s, ps = self.slab(lev), self.ps[lev]
        off = (s.plan.lo - s.e0) * ps
        cnt = s.plan.nplanes * ps
        xv, bv = self.ops.view(x, off, cnt), self.ops.view(b, off, cnt)
        SlabSmoother(s.plan, self.ops.kernel(lev, s.plan, xv, bv), self.comm(xv, ps)).smooth()

    def _gather_full(self, lev, a):
        """Owned planes of every rank -> the whole level vector."""
        s, ps = self.slab(lev), self.ps[lev]
        own = self.ops.view(a, (s.plan.own_lo - s.e0) * ps, (s.plan.own_hi - s.plan.own_lo + 1) * ps)
        return self.ops.cat(self.allgather(own))

    def vcycle(self, lev, x, b):
        s, ps = self.slab(lev), self.ps[lev]
        p = s.plan
        self._smooth(lev, x, b)
        self.halo(lev, x)
        self.ops.residual(lev, x, b, self.r[lev], s.e0, p.own_lo, p.own_hi + 1)
        self.halo(lev, self.r[lev])
        bc, xc = self.bc[lev], self.xc[lev]
        if lev - 1 in self.slabs:
            sc = self.slab(lev - 1)
            self.ops.restrict(lev, self.r[lev], s.e0, bc, sc.e0, sc.plan.own_lo, sc.plan.own_hi + 1)
            self.halo(lev - 1, bc)
            self.ops.fill(xc, 0.0)
            self.vcycle(lev - 1, xc, bc)
            self.halo(lev - 1, xc)
            e0c = sc.e0
        else:
            # agglomerated coarse level: this rank's share of R r, gathered,
            # then the rest of the V-cycle on the whole level (redundantly)
            mc = (1 << (lev - 1)) * self.k - 1
            q0, q1 = self._coarse_share(lev)
            self.ops.fill(bc, 0.0)
            self.ops.restrict(lev, self.r[lev], s.e0, bc, 0, q0, q1)
            part = self.ops.view(bc, q0 * self.ps[lev - 1], (q1 - q0) * self.ps[lev - 1])
            full_b = self.ops.cat(self.allgather(part))
            xfull = self.ops.vcycle_full(lev - 1, full_b)
            self.ops.copy(xc, xfull)
            e0c = 0
            del mc
        self.ops.prolongate(lev, xc, e0c, x, s.e0, p.lo, p.hi + 1)
        self._smooth(lev, x, b)

    def _coarse_share(self, lev):
        """Coarse planes this rank restricts at the agglomeration boundary: a
        contiguous partition of [0, mc) proportional to the fine ownership."""
        mc = (1 << (lev - 1)) * self.k - 1
        p = self.slab(lev).plan
        mf = p.mz
        q0 = 0 if self.rank == 0 else (p.own_lo * mc) // mf
        q1 = mc if self.rank == self.world - 1 else ((p.own_hi + 1) * mc) // mf
        return q0, q1


class GpuSlabOps:
    """SlabVCycle backend on the device: the C-ABI slab entry points of a
    MultigridContext (pmg.py) on CUDA tensors."""

    def __init__(self, mg, variant: str = "fused"):
        import torch

        from . import pmg as _pmg

        self.pmg, self.torch, self.mg, self.variant = _pmg, torch, mg, variant
        self.lv = {lc.level.level: lc for lc in mg.levels}
        self.dtype = torch.float64 if mg.levels[-1].dtype == np.float64 else torch.float32

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.dtype, device=f"cuda:{self.mg.device}")

    def view(self, a, off, cnt):
        return a[off:off + cnt]

    def fill(self, a, v):
        a.fill_(v)

    def cat(self, parts):
        return self.torch.cat(parts)

    def copy(self, dst, src):
        dst.copy_(src)

    def kernel(self, lev, plan, xv, bv):
        return gpu_kernel(self.lv[lev], plan, xv, bv, self.variant)

    def residual(self, lev, x, b, r, e0, p0, p1):
        self.pmg.compute_residual_slab(self.lv[lev], x, b, r, e0, p0, p1)

    def restrict(self, lev, rf, e0f, rc, e0c, q0, q1):
        self.pmg.restrict_slab(self.lv[lev - 1], self.lv[lev], rf, e0f, rc, e0c, q0, q1)

    def prolongate(self, lev, xc, e0c, xf, e0f, f0, f1):
        self.pmg.prolongate_slab(self.lv[lev - 1], self.lv[lev], xc, e0c, xf, e0f, f0, f1, True)

    def vcycle_full(self, lev, b):
        x = self.zeros(b.numel())
        self.pmg.v_cycle(self.mg, lev - 1, x, b)
        return x
