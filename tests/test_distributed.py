"""Row-partitioned aggregation and GCN epochs over 2-3 ranks with the gloo
backend on CPU.

Covers the multi-GPU host logic (edge-balanced row cut, padded-position
remap, the shift-pattern P2P stages, fp64 staged accumulation, the fp64
reduce-scatter backward through the reverse block, the replicated-weight GCN
epoch) with the CUDA row kernel replaced by an oracle stand-in inside the
worker processes that implements the same staged contract
(gmp_gspmm_staged: FIRST stores the fp64 partial, MID adds, LAST rounds once).
Results must equal the single-process full-graph oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1909_01315_b200 import distributed as D
from paper_1909_01315_b200 import generators
from paper_1909_01315_b200.graph import Graph


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_stage(block, x, rho, acc=None, mode=None, deg_full=None, out=None):
    """CPU stand-in for distributed.stage_aggregate (same staged contract)."""
    from oracle import gmp_oracle as O
    adj = block.to_csc()
    z, _ = O.gspmm(None, None, block.num_nodes, "copy_lhs", "src", None, "sum",
                   X=x.detach().to(torch.float64).numpy(),
                   adj=(adj.indptr.numpy(), adj.indices.numpy().astype(np.int64),
                        adj.edge_ids.numpy().astype(np.int64)))
    z = torch.from_numpy(z)
    deg = adj.degrees().to(torch.float64)
    if acc is None:
        if rho == "mean":
            z = z / deg.clamp_min(1).unsqueeze(1)
        return z.to(x.dtype)
    if mode & 1:
        z = z + acc
    if mode in (D.STAGE_FIRST, D.STAGE_MID):
        acc.copy_(z)
        return out
    if rho == "mean":
        dg = (deg_full if deg_full is not None else deg).to(torch.float64)
        z = z / dg.clamp_min(1).unsqueeze(1)
    out.copy_(z.to(out.dtype))
    return out


def _graph():
    s, d = generators.power_law_edges(400, 6, seed=3)
    return s, d, 400


def _worker(rank, world, port, results, dtype, rho, overlap):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    D.stage_aggregate = _oracle_stage  # CPU stand-in for the CUDA kernel
    s, d, n = _graph()
    g = Graph(s, d, n, device="cpu")
    pg = D.PartitionedGraph(g.to_csc(), n, rank, world)
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.standard_normal((n, 5)).astype(dtype))
    x_local = x[pg.r0:pg.r1].clone().requires_grad_(True)
    z_local = D.DistAggregate.apply(x_local, pg, overlap, rho)
    dz = torch.from_numpy(np.random.default_rng(1).standard_normal((n, 5)).astype(dtype))
    (z_local * dz[pg.r0:pg.r1]).sum().backward()
    results[rank] = (pg.r0, pg.r1, z_local.detach().numpy(), x_local.grad.numpy(),
                     int(pg.block.num_edges), len(pg.stage_blocks))
    dist.destroy_process_group()


def _run(world, dtype, rho, overlap):
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, port, results, dtype, rho, overlap), nprocs=world, join=True)
    return dict(results)


def test_partition_rows_balances_edges():
    indptr = np.concatenate([[0], np.cumsum([1000, 1, 1, 1, 500, 500, 1, 1])])
    b = D.partition_rows(indptr, 2)
    assert b[0] == 0 and b[-1] == 8 and np.all(np.diff(b) >= 0)
    edges = [indptr[b[i + 1]] - indptr[b[i]] for i in range(2)]
    assert max(edges) - min(edges) <= 1000
    b4 = D.partition_rows(np.arange(0, 101), 4)
    assert b4.tolist() == [0, 25, 50, 75, 100]


def test_stage_groups_cover_every_step_once():
    for world in (2, 3, 4, 8):
        for stages in (2, 3, 4, 9):
            groups = D.stage_groups(world, stages)
            flat = [k for gr in groups for k in gr]
            assert flat == list(range(1, world))
            assert len(groups) == min(stages - 1, world - 1)


def test_row_block_transpose_is_reverse():
    s, d, n = _graph()
    g = Graph(s, d, n, device="cpu")
    blk = D.RowBlock.rows_of(g.to_csc(), 0, n, n)
    rev = blk.transpose()
    csr = g.to_csr()
    assert torch.equal(rev.to_csc().indptr, csr.indptr)
    assert torch.equal(rev.to_csc().indices, csr.indices)
    assert torch.equal(rev.to_csc().edge_ids, csr.edge_ids)


def test_padded_positions_and_stage_blocks_partition_the_edges():
    """Every local edge lands in exactly one stage block; positions index the
    padded buffer at the owner's slot."""
    s, d, n = _graph()
    g = Graph(s, d, n, device="cpu")
    world = 4
    for rank in range(world):
        pg = D.PartitionedGraph(g.to_csc(), n, rank, world)
        w = pg.width
        pos = pg.block.to_csc().indices.to(torch.int64)
        owner = pos // w
        glob = torch.as_tensor(np.asarray(pg.bounds))[owner] + pos % w
        want = g.to_csc().indices[int(g.to_csc().indptr[pg.r0]):int(g.to_csc().indptr[pg.r1])]
        assert torch.equal(glob, want.to(torch.int64))
        total = pg.local_block.num_edges + sum(b.num_edges for b in pg.stage_blocks)
        assert total == pg.block.num_edges
        li = pg.local_block.to_csc().indices
        assert li.numel() == 0 or int(li.max()) < pg.num_local_rows


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("rho", ["sum", "mean"])
@pytest.mark.parametrize("overlap", [True, False])
def test_gloo_forward_backward_matches_single(world, rho, overlap):
    from oracle import gmp_oracle as O
    s, d, n = _graph()
    for dtype in (np.float64, np.float32):
        results = _run(world, dtype, rho, overlap)
        rng = np.random.default_rng(0)
        x = rng.standard_normal((n, 5)).astype(dtype).astype(np.float64)
        dz = np.random.default_rng(1).standard_normal((n, 5)).astype(dtype).astype(np.float64)
        want, _ = O.gspmm(s, d, n, "copy_lhs", "src", None, rho, X=x)
        want_dx = O.gspmm_backward(s, d, n, "copy_lhs", "src", None, rho, X=x, dZ=dz,
                                   aux=np.bincount(d, minlength=n))["src"]
        z = np.zeros_like(want)
        dx = np.zeros_like(want_dx)
        total_edges = 0
        for r in range(world):
            r0, r1, zl, dxl, ne, nst = results[r]
            z[r0:r1] = zl
            dx[r0:r1] = dxl
            total_edges += ne
            assert nst == min(2, world - 1)
        assert total_edges == len(s)
        if dtype == np.float64:
            assert np.allclose(z, want, rtol=1e-12, atol=1e-12)
            assert np.allclose(dx, want_dx, rtol=1e-12, atol=1e-12)
        else:  # fp32: one rounding of the fp64 sum - north_star's bar
            assert np.allclose(z, want, rtol=1e-5, atol=1e-6)
            assert np.allclose(dx, want_dx, rtol=1e-5, atol=1e-6)
            # staged fp64 accumulation rounds once: equals the rounded fp64 sum
            assert np.array_equal(z.astype(np.float32), want.astype(np.float32))


def _gcn_worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    D.stage_aggregate = _oracle_stage
    s, d, n = _graph()
    g = Graph(s, d, n, device="cpu")
    pg = D.PartitionedGraph(g.to_csc(), n, rank, world)
    rng = np.random.default_rng(2)
    x = torch.from_numpy(rng.standard_normal((n, 12)))
    labels = torch.from_numpy(rng.integers(0, 3, n))
    model = D.DistGCN([12, 8, 3], seed=0, aggregator="mean", device="cpu", dtype=torch.float64)
    losses = [float(model.train_epoch(pg, x[pg.r0:pg.r1], labels[pg.r0:pg.r1], 0.1))
              for _ in range(4)]
    results[rank] = (losses, [p.detach().numpy().copy() for p in model.parameters()])
    dist.destroy_process_group()


def test_gloo_gcn_epochs_match_across_world_sizes():
    """DistGCN's loss curve and weights on 2 and 3 ranks equal the 1-rank run
    (fp64): the partition, the staged forward and the reduce-scatter /
    all-reduce backward compose to the same full-graph gradient descent."""
    out = {}
    for world in (1, 2, 3):
        port = _free_port()
        mgr = mp.Manager()
        res = mgr.dict()
        mp.spawn(_gcn_worker, args=(world, port, res), nprocs=world, join=True)
        out[world] = dict(res)
    l1, p1 = out[1][0]
    for world in (2, 3):
        for r in range(world):
            lw, pw = out[world][r]
            assert np.allclose(lw, l1, rtol=1e-12, atol=1e-13), (world, lw, l1)
            for a, b in zip(pw, p1):
                assert np.allclose(a, b, rtol=1e-11, atol=1e-13)
    assert l1[-1] < l1[0]
