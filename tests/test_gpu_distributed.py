"""Row-partitioned aggregation on the GPU (distributed.py) through libgmp.

Single process: a rank's staged blocks (local shard first, then the shift
groups over the padded all-gather buffer, fp64-accumulated by
gmp_gspmm_staged) are run for every rank of a 3- and 8-way partition and
compared with the single-GPU g-SpMM: BIT-EXACT in fp32 (one rounding of the
same fp64 row sum) and for mean; the reverse blocks' fp64 partials summed
over ranks give dX. Two processes sharing cuda:0 (gloo carries the
collectives; NCCL refuses two ranks on one device) run DistAggregate and a
DistGCN epoch end to end. Wide rows (d = 602, unaligned ld) take the packed
column-tile path inside the blocks (tiles sized by source rows).
"""

import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import paper_1909_01315_b200 as G
from paper_1909_01315_b200 import distributed as D
from paper_1909_01315_b200 import kernels
from conftest import assert_close32, rel_err, to_np

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _padded(pg, x):
    buf = torch.zeros((pg.world * pg.width, x.shape[1]), dtype=x.dtype, device=x.device)
    for r in range(pg.world):
        b0, b1 = int(pg.bounds[r]), int(pg.bounds[r + 1])
        buf[r * pg.width:r * pg.width + (b1 - b0)] = x[b0:b1]
    return buf


def _staged(pg, x, rho):
    """What aggregate(overlap=True) computes, with every shard already landed."""
    xl = x[pg.r0:pg.r1].contiguous()
    acc = torch.empty((pg.num_local_rows, x.shape[1]), dtype=torch.float64, device=x.device)
    z = torch.empty((pg.num_local_rows, x.shape[1]), dtype=x.dtype, device=x.device)
    deg = pg.deg if rho == "mean" else None
    gathered = _padded(pg, x)
    D.stage_aggregate(pg.local_block, xl, rho, acc, D.STAGE_FIRST, deg, z)
    for i, blk in enumerate(pg.stage_blocks):
        last = i == len(pg.stage_blocks) - 1
        D.stage_aggregate(blk, gathered, rho, acc, D.STAGE_LAST if last else D.STAGE_MID, deg, z)
    return z


@pytest.mark.parametrize("world", [3, 8])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("F", [24, 602])
def test_staged_blocks_equal_single_gpu(world, dtype, F):
    n = 30000 if F == 602 else 3000
    s, d = G.generators.power_law_edges(n, 12, seed=0)
    g = G.from_arrays(s, d, num_nodes=n, device=DEV)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(0)
    x = torch.randn((n, F), generator=gen, device=DEV, dtype=dtype)
    bounds = D.partition_rows(g.to_csc().indptr, world)
    for rho in ("sum", "mean"):
        full, _ = G.gspmm(g, kernels.copy("src"), rho, X=x)
        for rank in range(world):
            pg = D.PartitionedGraph(g.to_csc(), n, rank, world, bounds=bounds)
            z_blk = D.local_aggregate(pg.block, _padded(pg, x), rho)
            z_st = _staged(pg, x, rho)
            want = full[pg.r0:pg.r1]
            if dtype == torch.float32:  # one rounding of the fp64 row sum: bit-exact
                assert torch.equal(z_blk, want), (rank, rho)
                assert torch.equal(z_st, want), (rank, rho)
            else:  # fp64 sums in another order
                assert rel_err(to_np(z_blk), to_np(want)) < 1e-13, (rank, rho)
                assert rel_err(to_np(z_st), to_np(want)) < 1e-13, (rank, rho)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_reverse_blocks_sum_to_dx(dtype):
    s, d = G.generators.power_law_edges(3000, 12, seed=1)
    n = 3000
    g = G.from_arrays(s, d, num_nodes=n, device=DEV)
    dz = torch.randn(n, 24, device=DEV, dtype=dtype)
    x = torch.randn(n, 24, device=DEV, dtype=dtype)
    want = G.gspmm_backward(g, kernels.copy("src"), "sum", X=x, dZ=dz, needs=("x",)).dx
    world = 3
    bounds = D.partition_rows(g.to_csc().indptr, world)
    total = None
    for rank in range(world):
        pg = D.PartitionedGraph(g.to_csc(), n, rank, world, bounds=bounds)
        rev = pg.reverse_block()
        part = torch.empty((rev.num_nodes, 24), dtype=torch.float64, device=DEV)
        D.stage_aggregate(rev, dz[pg.r0:pg.r1].contiguous(), "sum", part, D.STAGE_FIRST)
        total = part if total is None else total + part
    got = torch.cat([total[r * pg.width:r * pg.width + sz] for r, sz in enumerate(pg.sizes)])
    if dtype == torch.float64:
        assert rel_err(to_np(got), to_np(want)) < 1e-12
    else:
        assert_close32(got.float(), to_np(want).astype(np.float64), "dX")


def _mp_gpu_worker(rank, world, port, results, dtype):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s, d = G.generators.power_law_edges(3000, 12, seed=0)
    n = 3000
    g = G.from_arrays(s, d, num_nodes=n, device=DEV)
    pg = D.PartitionedGraph(g.to_csc(), n, rank, world)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(0)
    x = torch.randn((n, 16), generator=gen, device=DEV, dtype=dtype)
    dz = torch.randn((n, 16), generator=gen, device=DEV, dtype=dtype)
    out = {}
    for rho in ("sum", "mean"):
        x_local = x[pg.r0:pg.r1].clone().requires_grad_(True)
        z = D.DistAggregate.apply(x_local, pg, True, rho)
        (z * dz[pg.r0:pg.r1]).sum().backward()
        z_no = pg.aggregate(x[pg.r0:pg.r1].contiguous(), rho, overlap=False)
        out[rho] = (z.detach().cpu().numpy(), x_local.grad.cpu().numpy(), z_no.cpu().numpy())
    labels = torch.randint(0, 5, (n,), generator=gen, device=DEV)
    model = D.DistGCN([16, 8, 5], seed=0, aggregator="mean", device=DEV, dtype=dtype)
    losses = [float(model.train_epoch(pg, x[pg.r0:pg.r1], labels[pg.r0:pg.r1], 0.1))
              for _ in range(3)]
    torch.cuda.synchronize()
    results[rank] = (pg.r0, pg.r1, out, losses)
    dist.destroy_process_group()


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_two_process_row_partition_on_gpu(dtype):
    from paper_1909_01315_b200 import layers
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_mp_gpu_worker, args=(2, port, results, dtype), nprocs=2, join=True)
    s, d = G.generators.power_law_edges(3000, 12, seed=0)
    n = 3000
    g = G.from_arrays(s, d, num_nodes=n, device=DEV)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(0)
    x = torch.randn((n, 16), generator=gen, device=DEV, dtype=dtype)
    dz = torch.randn((n, 16), generator=gen, device=DEV, dtype=dtype)
    labels = torch.randint(0, 5, (n,), generator=gen, device=DEV)
    for rho in ("sum", "mean"):
        want, _ = G.gspmm(g, kernels.copy("src"), rho, X=x)
        bwd = G.gspmm_backward(g, kernels.copy("src"), rho, X=x, dZ=dz, needs=("x",),
                               aux=G.gspmm(g, kernels.copy("src"), rho, X=x)[1])
        want, want_dx = to_np(want), to_np(bwd.dx)
        for r in range(2):
            r0, r1, out, _ = results[r]
            z, dx, z_no = out[rho]
            if dtype == torch.float32:  # one rounding of the fp64 row sum: bit-exact
                assert np.array_equal(z, want[r0:r1]), rho
                assert np.array_equal(z_no, want[r0:r1]), rho
            else:
                assert rel_err(z, want[r0:r1]) < 1e-13 and rel_err(z_no, want[r0:r1]) < 1e-13
            if dtype == torch.float64:
                assert rel_err(dx, want_dx[r0:r1]) < 1e-12
            else:
                assert_close32(dx, want_dx[r0:r1].astype(np.float64), "dX " + rho)
    model = layers.GCNModel([16, 8, 5], seed=0, aggregator="mean", device=DEV, dtype=dtype)
    single = [float(layers.train_epoch(g, x, labels, model, 0.1)) for _ in range(3)]
    for r in range(2):
        tol = 1e-10 if dtype == torch.float64 else 1e-5
        assert np.allclose(results[r][3], single, rtol=tol, atol=tol), (results[r][3], single)
