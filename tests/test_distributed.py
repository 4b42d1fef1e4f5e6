"""Row-partitioned aggregation over 2 ranks with the gloo backend on CPU.

Covers the multi-GPU host logic (edge-balanced row cut, block construction,
padded all-gather, reduce-scatter backward through the reverse block) with
the CUDA row kernel replaced by the oracle inside the worker processes; the
result must equal the single-process full-graph oracle.
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


def _oracle_local_aggregate(block, x_full, rho="sum", out=None):
    from oracle import gmp_oracle as O
    adj = block.to_csc()
    z, _ = O.gspmm(None, None, block.num_nodes, "copy_lhs", "src", None, rho,
                   X=x_full.detach().numpy(),
                   adj=(adj.indptr.numpy(), adj.indices.numpy().astype(np.int64),
                        adj.edge_ids.numpy().astype(np.int64)))
    return torch.from_numpy(z).to(x_full.dtype)


def _graph():
    s, d = generators.power_law_edges(400, 6, seed=3)
    return s, d, 400


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    D.local_aggregate = _oracle_local_aggregate  # CPU stand-in for the CUDA kernel
    s, d, n = _graph()
    g = Graph(s, d, n, device="cpu")
    pg = D.PartitionedGraph(g.to_csc(), n, rank, world)
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.standard_normal((n, 5)))
    x_local = x[pg.r0:pg.r1].clone().requires_grad_(True)
    z_local = D.DistAggregate.apply(x_local, pg, False)
    dz = torch.from_numpy(np.random.default_rng(1).standard_normal((n, 5)))
    (z_local * dz[pg.r0:pg.r1]).sum().backward()
    results[rank] = (pg.r0, pg.r1, z_local.detach().numpy(), x_local.grad.numpy(),
                     int(pg.block.num_edges))
    dist.destroy_process_group()


def test_partition_rows_balances_edges():
    indptr = np.concatenate([[0], np.cumsum([1000, 1, 1, 1, 500, 500, 1, 1])])
    b = D.partition_rows(indptr, 2)
    assert b[0] == 0 and b[-1] == 8 and np.all(np.diff(b) >= 0)
    edges = [indptr[b[i + 1]] - indptr[b[i]] for i in range(2)]
    assert max(edges) - min(edges) <= 1000
    b4 = D.partition_rows(np.arange(0, 101), 4)
    assert b4.tolist() == [0, 25, 50, 75, 100]


def test_row_block_transpose_is_reverse():
    s, d, n = _graph()
    g = Graph(s, d, n, device="cpu")
    blk = D.RowBlock.rows_of(g.to_csc(), 0, n, n)
    rev = blk.transpose()
    csr = g.to_csr()
    assert torch.equal(rev.to_csc().indptr, csr.indptr)
    assert torch.equal(rev.to_csc().indices, csr.indices)
    assert torch.equal(rev.to_csc().edge_ids, csr.edge_ids)


def test_two_rank_gloo_forward_backward_matches_single():
    from oracle import gmp_oracle as O
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(2, port, results), nprocs=2, join=True)
    s, d, n = _graph()
    rng = np.random.default_rng(0)
    x = rng.standard_normal((n, 5))
    dz = np.random.default_rng(1).standard_normal((n, 5))
    want, _ = O.gspmm(s, d, n, "copy_lhs", "src", None, "sum", X=x)
    want_dx = O.gspmm_backward(s, d, n, "copy_lhs", "src", None, "sum", X=x, dZ=dz)["src"]
    z = np.zeros_like(want)
    dx = np.zeros_like(want_dx)
    total_edges = 0
    for r in range(2):
        r0, r1, zl, dxl, ne = results[r]
        z[r0:r1] = zl
        dx[r0:r1] = dxl
        total_edges += ne
    assert total_edges == len(s)
    assert np.allclose(z, want, rtol=1e-12, atol=1e-12)
    assert np.allclose(dx, want_dx, rtol=1e-12, atol=1e-12)
