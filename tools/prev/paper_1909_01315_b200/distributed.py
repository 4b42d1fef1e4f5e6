"""Destination-row partitioning across GPUs (one process per GPU, NCCL).

The north star's multi-GPU layout: the graph's CSC is cut into
contiguous destination-row ranges holding ~equal EDGE counts (cut on the
indptr prefix sum, so power-law hubs do not unbalance ranks - the
reference's node_parallel splits rows evenly instead, kernels.py:317-320,480).
Each rank owns the feature rows of its range.

Forward of one aggregation layer (`DistAggregate`):
  1. the row-sharded source features X are all-gathered over NCCL/NVLink
     (ranks may own different row counts: shards are padded to the largest);
  2. the row kernel runs on the local CSC block (global source ids, local
     destination rows). The output stays row-sharded and is the next layer's
     X shard, so no reduction is needed.
  With `overlap=True` the block is split by source owner: the part whose
  sources are local runs on the compute stream while the all-gather is in
  flight on a side stream, then the remote part accumulates into it.
Backward (Theorem 1 on a partition): each rank runs the reverse-graph row
kernel of its local block (rows = all n sources, local edges only) into a
full-length partial dX, then a reduce-scatter returns each rank its shard.

Host-side structures here are plain torch tensors; every aggregation goes
through `local_aggregate`, i.e. libgmp's row kernel.
"""

import itertools

import numpy as np
import torch

from .graph import Adjacency

_block_uid = itertools.count(10 ** 9)


def partition_rows(indptr, parts):
    """Row boundaries [0 = b0 <= ... <= b_parts = n] with ~m/parts edges each."""
    ip = indptr.cpu().numpy() if torch.is_tensor(indptr) else np.asarray(indptr)
    n = ip.size - 1
    m = int(ip[-1])
    targets = np.arange(1, parts, dtype=np.float64) * m / parts
    cuts = np.searchsorted(ip, targets, side="left").clip(0, n)
    bounds = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    return np.maximum.accumulate(bounds)


def shard_sizes(bounds):
    return [int(bounds[i + 1] - bounds[i]) for i in range(len(bounds) - 1)]


class RowBlock:
    """A grouped index over `num_nodes` rows whose neighbour ids index another
    node set (`num_src_nodes`) - the minimal graph view the row kernel
    launcher accepts (to_csc / num_nodes / device / uid)."""

    def __init__(self, indptr, indices, edge_ids, num_src_nodes):
        self._adj = Adjacency(indptr, indices, edge_ids)
        self.num_nodes = indptr.numel() - 1
        self.num_src_nodes = int(num_src_nodes)
        self.num_edges = indices.numel()
        self.device = indptr.device
        self.uid = next(_block_uid)

    def to_csc(self):
        return self._adj

    @classmethod
    def rows_of(cls, adj, r0, r1, num_src_nodes, keep=None):
        """Rows [r0, r1) of a CSC; `keep` optionally filters edges by a boolean
        mask over the block's neighbour ids (used to split by source owner)."""
        ip = adj.indptr[r0:r1 + 1]
        e0, e1 = int(ip[0]), int(ip[-1])
        ind = adj.indices[e0:e1]
        eid = adj.edge_ids[e0:e1]
        ip = ip - e0
        if keep is not None:
            sel = keep(ind)
            deg = torch.zeros(r1 - r0, dtype=torch.int64, device=ind.device)
            rows = torch.repeat_interleave(torch.arange(r1 - r0, device=ind.device),
                                           ip[1:] - ip[:-1])
            deg.index_add_(0, rows[sel], torch.ones_like(rows[sel]))
            ip = torch.zeros(r1 - r0 + 1, dtype=torch.int64, device=ind.device)
            torch.cumsum(deg, 0, out=ip[1:])
            ind, eid = ind[sel], eid[sel]
        return cls(ip, ind, eid, num_src_nodes)

    def transpose(self):
        """The reverse block: rows = source nodes (all num_src_nodes), neighbour
        ids = local destination rows; order (source, destination, edge id) as
        the reference's CSR (graph.py:35-44)."""
        dev = self.device
        rows = torch.repeat_interleave(torch.arange(self.num_nodes, device=dev),
                                       self._adj.indptr[1:] - self._adj.indptr[:-1])
        src = self._adj.indices.to(torch.int64)
        key = src * max(self.num_nodes, 1) + rows
        _, order = torch.sort(key, stable=True)
        counts = torch.bincount(src, minlength=self.num_src_nodes)
        ip = torch.zeros(self.num_src_nodes + 1, dtype=torch.int64, device=dev)
        torch.cumsum(counts, 0, out=ip[1:])
        return RowBlock(ip, rows.index_select(0, order).to(torch.int32),
                        self._adj.edge_ids.index_select(0, order), self.num_nodes)


def local_aggregate(block, x_full, rho="sum", out=None):
    """copy_u g-SpMM of a block's rows over source features x_full (libgmp)."""
    from . import kernels
    x_full = x_full.contiguous()
    z, _ = kernels._gspmm_launch(block, kernels.copy("src"), rho, x_full, None, None,
                                 x_full.shape[1], out=out)
    return z


def all_gather_rows(x_local, bounds, group=None, async_op=False):
    """Concatenate every rank's row shard; returns (tensor, work)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    sizes = shard_sizes(bounds)
    d = x_local.shape[1]
    width = max(sizes)
    if x_local.shape[0] == width:
        pad = x_local.contiguous()
    else:
        pad = torch.zeros((width, d), dtype=x_local.dtype, device=x_local.device)
        pad[:x_local.shape[0]] = x_local
    out = torch.empty((world * width, d), dtype=x_local.dtype, device=x_local.device)
    work = dist.all_gather_into_tensor(out, pad, group=group, async_op=async_op)
    return out, work, width


def unpad_rows(gathered, bounds, width):
    sizes = shard_sizes(bounds)
    if all(s == width for s in sizes):
        return gathered
    return torch.cat([gathered[r * width:r * width + s] for r, s in enumerate(sizes)])


def reduce_scatter_rows(partial, bounds, group=None):
    """Sum full-length (n, d) partials over ranks; return this rank's rows."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = shard_sizes(bounds)
    width = max(sizes)
    d = partial.shape[1]
    padded = torch.zeros((world * width, d), dtype=partial.dtype, device=partial.device)
    for r, s in enumerate(sizes):
        padded[r * width:r * width + s] = partial[int(bounds[r]):int(bounds[r]) + s]
    out = torch.empty((width, d), dtype=partial.dtype, device=partial.device)
    dist.reduce_scatter_tensor(out, padded, group=group)
    return out[:sizes[rank]]


class PartitionedGraph:
    """One rank's view of a destination-row-partitioned graph."""

    def __init__(self, adj, num_nodes, rank, world, bounds=None):
        self.num_nodes = int(num_nodes)
        self.rank, self.world = rank, world
        self.bounds = bounds if bounds is not None else partition_rows(adj.indptr, world)
        r0, r1 = int(self.bounds[rank]), int(self.bounds[rank + 1])
        self.r0, self.r1 = r0, r1
        self.block = RowBlock.rows_of(adj, r0, r1, num_nodes)
        # split by source owner: sources in [r0, r1) are local
        self.local_block = RowBlock.rows_of(adj, r0, r1, num_nodes,
                                            keep=lambda ind: (ind >= r0) & (ind < r1))
        self.remote_block = RowBlock.rows_of(adj, r0, r1, num_nodes,
                                             keep=lambda ind: (ind < r0) | (ind >= r1))
        self._rev = None

    @property
    def num_local_rows(self):
        return self.r1 - self.r0

    def reverse_block(self):
        if self._rev is None:
            self._rev = self.block.transpose()
        return self._rev

    def aggregate(self, x_local, rho="sum", overlap=False, group=None):
        """Forward g-SpMM (copy_u) of the local rows; x_local is this rank's shard."""
        if not overlap or self.world == 1:
            gathered, work, width = all_gather_rows(x_local, self.bounds, group)
            return local_aggregate(self.block, unpad_rows(gathered, self.bounds, width), rho)
        if rho != "sum":
            raise ValueError("overlapped aggregation supports rho='sum'")
        comm = torch.cuda.Stream(device=x_local.device)
        comm.wait_stream(torch.cuda.current_stream(x_local.device))
        with torch.cuda.stream(comm):
            gathered, work, width = all_gather_rows(x_local, self.bounds, group, async_op=True)
        # edges from local sources need no communication: run them first
        z = local_aggregate_offset(self.local_block, x_local, self.r0, rho)
        work.wait()
        torch.cuda.current_stream(x_local.device).wait_stream(comm)
        xf = unpad_rows(gathered, self.bounds, width)
        z += local_aggregate(self.remote_block, xf, rho)
        return z


def local_aggregate_offset(block, x_local, r0, rho="sum"):
    """Aggregate a block whose neighbour ids all lie in [r0, r0 + rows(x_local))
    reading only the local shard (neighbour ids rebased by -r0)."""
    ip = block.to_csc().indptr
    ind = (block.to_csc().indices - int(r0)).to(torch.int32)
    rebased = RowBlock(ip, ind, block.to_csc().edge_ids, x_local.shape[0])
    return local_aggregate(rebased, x_local, rho)


class DistAggregate(torch.autograd.Function):
    """Row-partitioned copy_u + sum with NCCL all-gather forward and
    reduce-scatter backward (dX through the reverse local block)."""

    @staticmethod
    def forward(ctx, x_local, pg, overlap):
        ctx.pg = pg
        return pg.aggregate(x_local, "sum", overlap=overlap)

    @staticmethod
    def backward(ctx, dz_local):
        pg = ctx.pg
        partial = local_aggregate(pg.reverse_block(), dz_local.contiguous(), "sum")
        return reduce_scatter_rows(partial, pg.bounds), None, None
