"""CPU: the multi-GPU slab decomposition's host logic (paper_2405_19004_b200/dd.py)
checked with the numpy oracle as the per-slab colour kernel, in one process
(virtual ranks) and across 2 processes over torch.distributed gloo."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import pmg_oracle as O
from paper_2405_19004_b200 import dd


def plans_for(world, k, level, stack):
    return [dd.make_plan(world, r, k, level, stack) for r in range(world)]


@pytest.mark.parametrize("world,k,level,stack", [(2, 2, 3, 1), (3, 1, 4, 1), (4, 3, 3, 1), (2, 2, 3, 2),
                                                 (4, 1, 2, 4), (8, 2, 3, 8), (5, 4, 3, 1)])
def test_plan_invariants(world, k, level, stack):
    ps = plans_for(world, k, level, stack)
    mz = ps[0].mz
    # owned planes partition [0, mz) and sit inside the local slabs
    assert ps[0].own_lo == 0 and ps[-1].own_hi == mz - 1
    for p, q in zip(ps, ps[1:]):
        assert p.own_hi + 1 == q.own_lo and p.b + 1 == q.a
    for p in ps:
        assert p.lo <= p.own_lo <= p.own_hi <= p.hi
        # the slab holds the closure of every owned patch (patches.cpp:71)
        assert p.lo <= max(0, k * (p.a - 1) - 1) and p.hi >= min(mz - 1, k * (p.b + 1) - 1)
    # every send has the matching receive on the peer, same planes
    for c in range(8):
        steps = [dd.colour_step(p, c) for p in ps]
        sends = {(r, q, g0, n) for r, s in enumerate(steps) for q, g0, n in s.sends}
        recvs = {(q, r, g0, n) for r, s in enumerate(steps) for q, g0, n in s.recvs}
        assert sends == recvs
        # one-directional per interface and colour
        for r in range(world - 1):
            ups = [s for s in sends if {s[0], s[1]} == {r, r + 1}]
            assert len(ups) <= 1


def oracle_kernel(ctx, plan, x_loc, b_loc):
    def run(color, vlo, vhi):
        O.smooth_colour_slab(ctx, x_loc, b_loc, color, plan.lo, plan.nz, vlo, vhi)
    return run


@pytest.mark.parametrize("world,k,level", [(2, 2, 3), (3, 1, 4), (4, 3, 3), (2, 4, 2), (7, 1, 3)])
def test_virtual_slabs_equal_full_smooth(world, k, level):
    """P slabs of the unit cube == the oracle's single-domain smooth."""
    ctx = O.MultigridContext(3, k, level)
    lc = ctx.levels[-1]
    rng = np.random.default_rng(11)
    x0 = rng.uniform(-1, 1, lc.level.total_dofs)
    b = rng.uniform(-1, 1, lc.level.total_dofs)
    want = O.smooth(lc, x0, b)
    ps = plans_for(world, k, level, 1)
    xs = [dd.scatter_global(p, x0).copy() for p in ps]
    bs = [dd.scatter_global(p, b).copy() for p in ps]
    dd.virtual_smooth(ps, [oracle_kernel(lc, p, x, bb) for p, x, bb in zip(ps, xs, bs)], xs)
    got = np.concatenate([dd.owned_part(p, x) for p, x in zip(ps, xs)])
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-13 * np.abs(want).max())


def test_virtual_stacked_box_matches_one_rank():
    """Weak-scaling geometry (stack = world cubes along z): P slabs == 1 slab."""
    k, level, world = 2, 3, 4
    lc = O.MultigridContext(3, k, level).levels[-1]
    p1 = dd.make_plan(1, 0, k, level, world)
    rng = np.random.default_rng(12)
    n = p1.nplanes * p1.plane_size
    x0, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    x1 = x0.copy()
    dd.virtual_smooth([p1], [oracle_kernel(lc, p1, x1, b)], [x1])
    ps = plans_for(world, k, level, world)
    xs = [dd.scatter_global(p, x0).copy() for p in ps]
    bs = [dd.scatter_global(p, b).copy() for p in ps]
    dd.virtual_smooth(ps, [oracle_kernel(lc, p, x, bb) for p, x, bb in zip(ps, xs, bs)], xs)
    got = np.concatenate([dd.owned_part(p, x) for p, x in zip(ps, xs)])
    np.testing.assert_allclose(got, x1, rtol=0, atol=1e-13 * np.abs(x1).max())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, k, level, stack, out_path):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lc = O.MultigridContext(3, k, level).levels[-1]
        plan = dd.make_plan(world, rank, k, level, stack)
        full = dd.make_plan(1, 0, k, level, stack)
        rng = np.random.default_rng(21)
        n = full.nplanes * full.plane_size
        x0, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        xt = torch.from_numpy(dd.scatter_global(plan, x0).copy())
        bl = dd.scatter_global(plan, b).copy()
        sm = dd.SlabSmoother(plan, oracle_kernel(lc, plan, xt.numpy(), bl), dd.TorchDistComm(xt, plan.plane_size))
        sm.smooth()
        own = torch.from_numpy(dd.owned_part(plan, xt.numpy()).copy())
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([own.numel()]))
        mx = int(max(s.item() for s in sizes))
        padded = torch.zeros(mx, dtype=own.dtype)
        padded[: own.numel()] = own
        parts = [torch.zeros(mx, dtype=own.dtype) for _ in sizes]
        dist.all_gather(parts, padded)
        if rank == 0:
            got = torch.cat([p[: int(s.item())] for p, s in zip(parts, sizes)]).numpy()
            x1 = x0.copy()
            dd.virtual_smooth([full], [oracle_kernel(lc, full, x1, b)], [x1])
            np.save(out_path, np.array([np.abs(got - x1).max(), np.abs(x1).max()]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("stack", [1, 2])
def test_gloo_two_ranks(tmp_path, stack):
    """world_size 2 over gloo (the GPU path uses the same driver over NCCL)."""
    out = str(tmp_path / "err.npy")
    mp.spawn(_gloo_worker, args=(2, _free_port(), 2, 3, stack, out), nprocs=2, join=True)
    err, scale = np.load(out)
    assert err <= 1e-13 * scale


# ---------------------------------------------------------------------------
# The slab-decomposed V-cycle (dd.SlabVCycle) with the numpy oracle as the
# backend: P ranks over gloo == the oracle's single-domain V-cycle.
# ---------------------------------------------------------------------------


class OracleSlabOps:
    """dd.SlabVCycle backend on the CPU: every slab operation embeds the slab
    into a zero global vector, applies the oracle's full-domain operation and
    keeps the requested planes (which only depend on planes the slab holds)."""

    def __init__(self, octx):
        self.o = octx
        self.lc = {lc.level.level: lc for lc in octx.levels}

    def ps(self, lev):
        return self.lc[lev].level.dofs_per_dim ** 2

    def embed(self, lev, a, e0):
        full = np.zeros(self.lc[lev].level.total_dofs)
        full[e0 * self.ps(lev):e0 * self.ps(lev) + a.size] = a
        return full

    def zeros(self, n):
        return np.zeros(n)

    def view(self, a, off, cnt):
        return a[off:off + cnt]

    def fill(self, a, v):
        a[:] = v

    def cat(self, parts):
        return np.concatenate([np.asarray(p) for p in parts])

    def copy(self, dst, src):
        dst[:] = src

    def kernel(self, lev, plan, xv, bv):
        lc = self.lc[lev]
        return lambda c, vlo, vhi: O.smooth_colour_slab(lc, xv, bv, c, plan.lo, plan.nz, vlo, vhi)

    def residual(self, lev, x, b, r, e0, p0, p1):
        ps = self.ps(lev)
        rf = O.compute_residual(self.lc[lev], self.embed(lev, x, e0), self.embed(lev, b, e0))
        r[(p0 - e0) * ps:(p1 - e0) * ps] = rf[p0 * ps:p1 * ps]

    def restrict(self, lev, rf, e0f, rc, e0c, q0, q1):
        psc = self.ps(lev - 1)
        full = O.restrict_vector(self.lc[lev - 1], self.lc[lev], self.embed(lev, rf, e0f))
        rc[(q0 - e0c) * psc:(q1 - e0c) * psc] = full[q0 * psc:q1 * psc]

    def prolongate(self, lev, xc, e0c, xf, e0f, f0, f1):
        ps = self.ps(lev)
        full = O.prolongate(self.lc[lev - 1], self.lc[lev], self.embed(lev - 1, xc, e0c))
        xf[(f0 - e0f) * ps:(f1 - e0f) * ps] += full[f0 * ps:f1 * ps]

    def vcycle_full(self, lev, b):
        return O.v_cycle(self.o, lev - 1, np.zeros_like(b), b)


def _gloo_vcycle_worker(rank, world, port, k, level, out_path):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        octx = O.MultigridContext(3, k, level)
        n = octx.levels[-1].level.total_dofs
        rng = np.random.default_rng(31)
        x0, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)

        def comm(a, ps):
            return dd.TorchDistComm(torch.from_numpy(a), ps)

        def allgather(part):
            t = torch.from_numpy(np.ascontiguousarray(part))
            sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(sizes, torch.tensor([t.numel()]))
            mx = int(max(s.item() for s in sizes))
            padded = torch.zeros(mx, dtype=t.dtype)
            padded[: t.numel()] = t
            parts = [torch.zeros(mx, dtype=t.dtype) for _ in sizes]
            dist.all_gather(parts, padded)
            return [p[: int(s.item())].numpy() for p, s in zip(parts, sizes)]

        vc = dd.SlabVCycle(world, rank, k, level, OracleSlabOps(octx), comm, allgather)
        s = vc.slab(level)
        ps = s.plan.plane_size
        x = x0[s.e0 * ps:(s.e1 + 1) * ps].copy()
        bl = b[s.e0 * ps:(s.e1 + 1) * ps].copy()
        vc.vcycle(level, x, bl)
        own = x[(s.plan.own_lo - s.e0) * ps:(s.plan.own_hi - s.e0 + 1) * ps]
        got = np.concatenate(allgather(own))
        if rank == 0:
            want = O.v_cycle(octx, level - 1, x0.copy(), b)
            np.save(out_path, np.array([np.abs(got - want).max(), np.abs(want).max(), vc.agg]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k,level", [(2, 1, 6), (2, 2, 5), (3, 1, 6)])
def test_gloo_slab_vcycle(tmp_path, world, k, level):
    """The slab-decomposed V-cycle over gloo == the single-domain V-cycle."""
    out = str(tmp_path / "err.npy")
    mp.spawn(_gloo_vcycle_worker, args=(world, _free_port(), k, level, out), nprocs=world, join=True)
    err, scale, agg = np.load(out)
    assert agg >= 1
    assert err <= 1e-13 * scale, (err, scale)


# ---------------------------------------------------------------------------
# The C++ decomposition (csrc/dd.cu, pmg_dd_*) follows the same plan as this
# module: compare the host-only plan dump with make_plan / colour_step /
# decomposed_levels over many (world, rank, k, level, stack). No GPU needed.
# ---------------------------------------------------------------------------
import ctypes  # noqa: E402


def _cpp_plan(world, rank, k, level, stack):
    from paper_2405_19004_b200 import _lib

    buf = (ctypes.c_int64 * 4096)()
    n = _lib.load().pmg_dd_plan(world, rank, k, level, stack, buf, 4096)
    assert n > 0, n
    v = list(buf[:n])
    head, rest = v[:7], v[7:]
    steps = []
    for _ in range(8):
        ne, ns, nr = rest[:3]
        rest = rest[3:]
        early = rest[:ne]
        rest = rest[ne:]
        sends = [tuple(rest[3 * i:3 * i + 3]) for i in range(ns)]
        rest = rest[3 * ns:]
        recvs = [tuple(rest[3 * i:3 * i + 3]) for i in range(nr)]
        rest = rest[3 * nr:]
        steps.append((early, sends, recvs))
    return head, steps


@pytest.mark.parametrize("world", [1, 2, 3, 4, 7, 8])
@pytest.mark.parametrize("k,level,stack", [(1, 4, 1), (2, 5, 1), (3, 4, 1), (4, 6, 1), (7, 3, 1), (2, 4, 4),
                                           (3, 3, 8)])
def test_cpp_plan_matches_python(world, k, level, stack):
    from paper_2405_19004_b200 import dd

    if (1 << level) * stack - 1 < world:
        return
    dl = dd.decomposed_levels(world, k, level) if stack == 1 else []
    for rank in range(world):
        p = dd.make_plan(world, rank, k, level, stack=stack)
        head, steps = _cpp_plan(world, rank, k, level, stack)
        assert head == [p.a, p.b, p.lo, p.hi, p.own_lo, p.own_hi, int(level in dl)]
        for c in range(8):
            st = dd.colour_step(p, c)
            assert steps[c][0] == [lo for lo, _ in st.early]
            assert steps[c][1] == [tuple(m) for m in st.sends]
            assert steps[c][2] == [tuple(m) for m in st.recvs]


def test_cpp_plan_errors():
    from paper_2405_19004_b200 import _lib

    buf = (ctypes.c_int64 * 16)()
    assert _lib.load().pmg_dd_plan(8, 0, 2, 2, 1, buf, 16) < 0  # 3 vertex planes over 8 ranks
    assert _lib.load().pmg_dd_plan(2, 0, 2, 5, 1, buf, 4) < 0   # capacity


# ---------------------------------------------------------------------------
# SURVEY.md §8e alternative: one exchange per step with an 8-vertex-plane
# halo and redundant halo patches (dd.DeepHaloSmoother) == one domain.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("world,k,level,steps", [(2, 2, 4, 2), (3, 1, 5, 3), (2, 3, 4, 1), (4, 1, 5, 2), (5, 2, 3, 2)])
def test_virtual_deep_halo_equals_full_smooth(world, k, level, steps):
    ctx = O.MultigridContext(3, k, level)
    lc = ctx.levels[-1]
    rng = np.random.default_rng(5)
    x0 = rng.uniform(-1, 1, lc.level.total_dofs)
    b = rng.uniform(-1, 1, lc.level.total_dofs)
    want = x0.copy()
    for _ in range(steps):
        want = O.smooth(lc, want, b)
    ps = [dd.deep_halo_plan(p) for p in plans_for(world, k, level, 1)]
    xs = [dd.scatter_global(p, x0).copy() for p in ps]
    bs = [dd.scatter_global(p, b).copy() for p in ps]
    for _ in range(steps):
        dd.virtual_deep_smooth(ps, [oracle_kernel(lc, p, x, bb) for p, x, bb in zip(ps, xs, bs)], xs)
    got = np.concatenate([dd.owned_part(p, x) for p, x in zip(ps, xs)])
    np.testing.assert_array_equal(got, want)


def _gloo_deep_worker(rank, world, port, k, level, out_path):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lc = O.MultigridContext(3, k, level).levels[-1]
        plans = [dd.deep_halo_plan(dd.make_plan(world, r, k, level)) for r in range(world)]
        plan = plans[rank]
        sends, recvs = dd.deep_halo_messages(plans)[rank]
        full = dd.make_plan(1, 0, k, level)
        rng = np.random.default_rng(23)
        n = full.nplanes * full.plane_size
        x0, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        xt = torch.from_numpy(dd.scatter_global(plan, x0).copy())
        bl = dd.scatter_global(plan, b).copy()
        sm = dd.DeepHaloSmoother(plan, sends, recvs, oracle_kernel(lc, plan, xt.numpy(), bl),
                                 dd.TorchDistComm(xt, plan.plane_size))
        for _ in range(2):
            sm.smooth()
        own = torch.from_numpy(dd.owned_part(plan, xt.numpy()).copy())
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([own.numel()]))
        mx = int(max(s.item() for s in sizes))
        padded = torch.zeros(mx, dtype=own.dtype)
        padded[: own.numel()] = own
        parts = [torch.zeros(mx, dtype=own.dtype) for _ in sizes]
        dist.all_gather(parts, padded)
        if rank == 0:
            got = torch.cat([p[: int(s.item())] for p, s in zip(parts, sizes)]).numpy()
            want = x0.copy()
            for _ in range(2):
                want = O.smooth(lc, want, b)
            np.save(out_path, np.array([float(np.abs(got - want).max())]))
    finally:
        dist.destroy_process_group()


def test_gloo_deep_halo_three_ranks(tmp_path):
    """The single-exchange step over torch.distributed (gloo, world 3)."""
    out = str(tmp_path / "err.npy")
    mp.spawn(_gloo_deep_worker, args=(3, _free_port(), 2, 4, out), nprocs=3, join=True)
    assert np.load(out)[0] == 0.0
