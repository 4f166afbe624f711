"""GPU: the slab-decomposed V-cycle (paper_2405_19004_b200/dd.py SlabVCycle)
with the device slab kernels (pmg_compute_residual_slab, pmg_restrict_slab,
pmg_prolongate_slab, pmg_smooth_color_slab): P ranks (processes sharing the
one GPU of this box, gloo with host-staged plane messages) reproduce the
single-GPU V-cycle bitwise. On an 8-GPU box the same driver runs over NCCL."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, k, level, dtype, out_path):
    import torch
    import torch.distributed as dist

    import paper_2405_19004_b200 as pmg
    from paper_2405_19004_b200 import dd

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        npdt = np.float64 if dtype == "f64" else np.float32
        tdt = torch.float64 if dtype == "f64" else torch.float32
        mg = pmg.make_multigrid_context(3, k, level, dtype=npdt)
        n = mg.levels[-1].level.total_dofs
        rng = np.random.default_rng(41)
        x0 = torch.from_numpy(rng.uniform(-1, 1, n).astype(npdt)).cuda()
        b = torch.from_numpy(rng.uniform(-1, 1, n).astype(npdt)).cuda()

        def comm(a, ps):
            return dd.StagedComm(a, ps)

        def allgather(part):
            t = part.detach().cpu().contiguous()
            sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(sizes, torch.tensor([t.numel()]))
            mx = int(max(s.item() for s in sizes))
            padded = torch.zeros(mx, dtype=t.dtype)
            padded[: t.numel()] = t
            parts = [torch.zeros(mx, dtype=t.dtype) for _ in sizes]
            dist.all_gather(parts, padded)
            return [p[: int(s.item())].cuda() for p, s in zip(parts, sizes)]

        vc = dd.SlabVCycle(world, rank, k, level, dd.GpuSlabOps(mg), comm, allgather)
        s = vc.slab(level)
        ps = s.plan.plane_size
        x = x0[s.e0 * ps:(s.e1 + 1) * ps].clone()
        bl = b[s.e0 * ps:(s.e1 + 1) * ps].clone()
        for _ in range(2):
            vc.vcycle(level, x, bl)
        own = x[(s.plan.own_lo - s.e0) * ps:(s.plan.own_hi - s.e0 + 1) * ps]
        got = torch.cat(allgather(own)).cpu().numpy()
        if rank == 0:
            want = x0.clone()
            for _ in range(2):
                pmg.v_cycle(mg, level - 1, want, b)
            want = want.cpu().numpy()
            np.save(out_path, np.array([float(np.array_equal(got, want)), np.abs(got - want).max(),
                                        np.abs(want).max(), vc.agg]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k,level,dtype", [(2, 1, 6, "f64"), (2, 1, 7, "f64"), (2, 2, 5, "f64"),
                                                 (3, 2, 6, "f32"), (4, 2, 6, "f64"), (2, 3, 5, "f64"),
                                                 (2, 4, 5, "f64")])
def test_slab_vcycle_bitwise(tmp_path, world, k, level, dtype):
    out = str(tmp_path / "res.npy")
    mp.spawn(_worker, args=(world, _free_port(), k, level, dtype, out), nprocs=world, join=True)
    same, err, scale, agg = np.load(out)
    assert same == 1.0, (err, scale, agg)


def _smoother_worker(rank, world, port, k, level, stack, out_path):
    import torch
    import torch.distributed as dist

    import paper_2405_19004_b200 as pmg
    from paper_2405_19004_b200 import dd

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        mg = pmg.make_multigrid_context(3, k, level, dtype=np.float64)
        lev = mg.levels[-1]
        full = dd.make_plan(1, 0, k, level, stack)
        n = full.nplanes * full.plane_size
        rng = np.random.default_rng(51)
        x0 = torch.from_numpy(rng.uniform(-1, 1, n)).cuda()
        b = torch.from_numpy(rng.uniform(-1, 1, n)).cuda()
        plan = dd.make_plan(world, rank, k, level, stack)
        x = dd.scatter_global(plan, x0).clone()
        bl = dd.scatter_global(plan, b).clone()
        sm = dd.SlabSmoother(plan, dd.gpu_kernel(lev, plan, x, bl), dd.StagedComm(x, plan.plane_size),
                             side_stream=torch.cuda.Stream())
        for _ in range(2):
            sm.smooth()
        torch.cuda.synchronize()
        own = dd.owned_part(plan, x).cpu()
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([own.numel()]))
        mx = int(max(s.item() for s in sizes))
        padded = torch.zeros(mx, dtype=own.dtype)
        padded[: own.numel()] = own
        parts = [torch.zeros(mx, dtype=own.dtype) for _ in sizes]
        dist.all_gather(parts, padded)
        if rank == 0:
            got = torch.cat([p[: int(s.item())] for p, s in zip(parts, sizes)]).numpy()
            xg = x0.clone()
            for _ in range(2):
                dd.virtual_smooth([full], [dd.gpu_kernel(lev, full, xg, b)], [xg])
            want = xg.cpu().numpy()
            np.save(out_path, np.array([float(np.array_equal(got, want)), np.abs(got - want).max()]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k,level,stack", [(2, 2, 5, 1), (2, 3, 4, 2), (3, 2, 4, 3)])
def test_slab_smoother_side_stream_bitwise(tmp_path, world, k, level, stack):
    """SlabSmoother with the boundary-layer patches and plane messages on a
    side stream (the NCCL bench path's organisation) == one domain, bitwise."""
    out = str(tmp_path / "res.npy")
    mp.spawn(_smoother_worker, args=(world, _free_port(), k, level, stack, out), nprocs=world, join=True)
    same, err = np.load(out)
    assert same == 1.0, err
