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
