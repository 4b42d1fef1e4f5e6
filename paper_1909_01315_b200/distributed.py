"""Destination-row partitioning across GPUs (one process per GPU, NCCL).

The north star's multi-GPU layout: the graph's CSC is cut into
contiguous destination-row ranges holding ~equal EDGE counts (cut on the
indptr prefix sum, so power-law hubs do not unbalance ranks - the
reference's node_parallel splits rows evenly instead, kernels.py:317-320,480).
Each rank owns the feature rows of its range. A g-SpMM layer then:
  1. all-gathers the row-sharded source features X over NCCL / NVLink,
  2. runs the row kernel on its local CSC block (global source ids,
     local destination rows) - the output stays row-sharded and is the next
     layer's X shard, so no reduction is needed.
Backward dX is the reverse-graph kernel on the local block into a full-length
partial followed by a reduce-scatter (not needed by the forward bench).

`RowBlock` is a minimal graph view the kernel launcher accepts: it exposes the
local CSC and the row count, nothing else.
"""

import itertools

import numpy as np
import torch

from .graph import Adjacency

_block_uid = itertools.count(10 ** 9)


def partition_rows(indptr, parts):
    """Row boundaries [b0=0, ..., b_parts=n] with ~m/parts edges per range."""
    ip = indptr.cpu().numpy() if torch.is_tensor(indptr) else np.asarray(indptr)
    n = ip.size - 1
    m = int(ip[-1])
    targets = (np.arange(1, parts, dtype=np.float64) * m / parts)
    cuts = np.searchsorted(ip, targets, side="left").clip(0, n)
    bounds = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    return np.maximum.accumulate(bounds)


class RowBlock:
    """Rows [r0, r1) of a CSC with global neighbour ids."""

    def __init__(self, adj, r0, r1, num_src_nodes):
        ip = adj.indptr[r0:r1 + 1]
        e0, e1 = int(ip[0]), int(ip[-1])
        self._adj = Adjacency(ip - e0, adj.indices[e0:e1], adj.edge_ids[e0:e1])
        self.r0, self.r1 = int(r0), int(r1)
        self.num_src_nodes = int(num_src_nodes)
        self.num_nodes = self.r1 - self.r0
        self.num_edges = e1 - e0
        self.device = adj.indptr.device
        self.uid = next(_block_uid)

    def to_csc(self):
        return self._adj


def shard_sizes(bounds):
    return [int(bounds[i + 1] - bounds[i]) for i in range(len(bounds) - 1)]


def all_gather_rows(x_local, bounds, group=None):
    """Concatenate every rank's row shard (ranks may own different row counts)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    sizes = shard_sizes(bounds)
    d = x_local.shape[1]
    width = max(sizes)
    pad = torch.zeros((width, d), dtype=x_local.dtype, device=x_local.device)
    pad[:x_local.shape[0]] = x_local
    out = torch.empty((world * width, d), dtype=x_local.dtype, device=x_local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    if all(s == width for s in sizes):
        return out
    return torch.cat([out[r * width:r * width + sizes[r]] for r in range(world)])


def local_aggregate(block, x_full, rho="sum"):
    """copy_u g-SpMM of one rank's rows over the gathered source features."""
    from . import kernels
    x_full = x_full.contiguous()
    phi = kernels.copy("src")
    z, _ = kernels._gspmm_launch(block, phi, rho, x_full, None, None, x_full.shape[1])
    return z
