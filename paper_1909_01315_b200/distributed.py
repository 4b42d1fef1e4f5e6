"""Destination-row partitioning across GPUs (one process per GPU, NCCL).

The north star's multi-GPU layout: the graph's CSC is cut into
contiguous destination-row ranges holding ~equal EDGE counts (cut on the
indptr prefix sum, so power-law hubs do not unbalance ranks - the
reference's node_parallel splits rows evenly instead, kernels.py:317-320,480).
Each rank owns the feature rows of its range.

Layout. Shards are gathered into one padded buffer, rank r's rows at
[r * width, r * width + size_r) with width = the largest shard. Every block's
neighbour ids are remapped at partition time to positions in that buffer, so
the row kernel gathers straight out of it (no un-padding copy), and the
reverse block's rows are those positions, so the backward's full-length
partial IS the reduce-scatter input.

Forward of one aggregation (`aggregate`, `DistAggregate`):
  stage 0  the edges whose sources this rank owns, read from the local shard
           (no communication), run while the other shards are in flight;
  stage s  the edges whose sources arrived in step group s. Shards move by a
           shift pattern over NVSwitch: at step k every rank sends its shard
           to rank + k and receives rank - k's (NCCL P2P on a side stream;
           every GPU pair has full bandwidth, so no ring forwarding), and a
           group's block runs as soon as its shards have landed.
  The stages accumulate into ONE fp64 row buffer (gmp_gspmm_staged) and round
  once at the last stage: the same single rounding as one kernel over the
  whole row (the reference sums each row in float64, kernels.py:396). Z stays
  row-sharded and is the next layer's X shard.
Backward (Theorem 1 on a partition): the reverse block (rows = padded source
positions, local edges only) aggregates dZ into an fp64 full-length partial,
NCCL reduce-scatter sums the ranks' partials in fp64, and each rank rounds its
shard once.

Every aggregation goes through `stage_aggregate` (libgmp's row kernel).
"""

import itertools

import numpy as np
import torch

from .graph import Adjacency

_block_uid = itertools.count(10 ** 9)

STAGE_FIRST, STAGE_MID, STAGE_LAST = 0, 1, 3  # gmp.h GMP_STAGE_*


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


def stage_groups(world, stages):
    """Shift steps 1..world-1 split into (stages - 1) contiguous groups; stage
    0 (the local shard) needs no step."""
    steps = list(range(1, world))
    groups = max(1, min(stages - 1, len(steps)))
    return [list(c) for c in np.array_split(np.array(steps, dtype=np.int64), groups) if len(c)]


class RowBlock:
    """A grouped index over `num_nodes` rows whose neighbour ids index another
    node set (`num_src_nodes`) - the minimal graph view the row kernel
    launcher accepts (to_csc / num_nodes / device / uid). Its schedule is
    built once (the block is cached by its PartitionedGraph)."""

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
    def rows_of(cls, adj, r0, r1, num_src_nodes, keep=None, remap=None):
        """Rows [r0, r1) of a CSC. `keep` filters edges by a boolean mask over
        the neighbour ids; `remap` maps the kept neighbour ids to the ids the
        block gathers with (e.g. positions in the padded all-gather buffer)."""
        ip = adj.indptr[r0:r1 + 1]
        e0, e1 = int(ip[0]), int(ip[-1])
        ind = adj.indices[e0:e1]
        eid = adj.edge_ids[e0:e1]
        ip = ip - e0
        if keep is not None:
            sel = keep(ind)
            rows = torch.repeat_interleave(torch.arange(r1 - r0, device=ind.device),
                                           ip[1:] - ip[:-1])
            deg = torch.bincount(rows[sel], minlength=r1 - r0)
            ip = torch.zeros(r1 - r0 + 1, dtype=torch.int64, device=ind.device)
            torch.cumsum(deg, 0, out=ip[1:])
            ind, eid = ind[sel], eid[sel]
        if remap is not None:
            ind = remap(ind).to(torch.int32)
        return cls(ip, ind.contiguous(), eid.contiguous(), num_src_nodes)

    def transpose(self):
        """The reverse block: rows = the source ids (all num_src_nodes),
        neighbour ids = local destination rows; order (source, destination,
        edge id) as the reference's CSR (graph.py:35-44)."""
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


def stage_aggregate(block, x, rho, acc=None, mode=None, deg_full=None, out=None):
    """copy_u sum / mean of a block's rows over source rows x (libgmp). With
    acc / mode: one stage of an fp64-accumulated staged sum
    (gmp_gspmm_staged); Z (out) is written by the STAGE_LAST launch only."""
    from . import kernels
    x = x.contiguous()
    if acc is None:
        z, _ = kernels._gspmm_launch(block, kernels.copy("src"), rho, x, None, None,
                                     x.shape[1], out=out)
        return z
    if out is None:
        out = torch.empty((block.num_nodes, x.shape[1]), dtype=x.dtype, device=x.device)
    kernels._gspmm_launch(block, kernels.copy("src"), rho, x, None, None, x.shape[1], out=out,
                          stage=(acc, mode, deg_full))
    return out


def local_aggregate(block, x_full, rho="sum", out=None):
    """copy_u g-SpMM of a block's rows over source features x_full (libgmp)."""
    return stage_aggregate(block, x_full, rho, out=out)


def _is_nccl(group=None):
    import torch.distributed as dist
    return dist.get_backend(group) == "nccl"


class PartitionedGraph:
    """One rank's view of a destination-row-partitioned graph. Built once:
    the blocks (with their row schedules) are cached, nothing is rebuilt per
    step."""

    def __init__(self, adj, num_nodes, rank, world, bounds=None, stages=3):
        self.num_nodes = int(num_nodes)
        self.rank, self.world = rank, world
        self.bounds = bounds if bounds is not None else partition_rows(adj.indptr, world)
        self.sizes = shard_sizes(self.bounds)
        self.width = max(max(self.sizes), 1)
        r0, r1 = int(self.bounds[rank]), int(self.bounds[rank + 1])
        self.r0, self.r1 = r0, r1
        dev = adj.indptr.device
        bt = torch.as_tensor(np.asarray(self.bounds), dtype=torch.int64, device=dev)
        width = self.width

        def owner(ind):
            return torch.searchsorted(bt, ind.to(torch.int64), right=True) - 1

        def padded(ind):  # global id -> row of the padded gathered buffer
            o = owner(ind)
            return o * width + (ind.to(torch.int64) - bt[o])

        self._owner = owner
        P = world * width
        # whole local block over the padded buffer (non-overlapped path, backward)
        self.block = RowBlock.rows_of(adj, r0, r1, P, remap=padded)
        self.deg = self.block.to_csc().degrees().clone()
        # stage 0: local sources, read from the local shard itself
        self.local_block = RowBlock.rows_of(
            adj, r0, r1, r1 - r0, keep=lambda ind: owner(ind) == rank,
            remap=lambda ind: ind.to(torch.int64) - r0)
        # remote stages: sources owned by the ranks the shift steps of a group reach
        self.groups = stage_groups(world, stages) if world > 1 else []
        self.stage_blocks = []
        for steps in self.groups:
            owners = torch.as_tensor([(rank - k) % world for k in steps], device=dev)
            self.stage_blocks.append(RowBlock.rows_of(
                adj, r0, r1, P, keep=lambda ind, o=owners: torch.isin(owner(ind), o),
                remap=padded))
        if dev.type == "cuda":  # row schedules built once, outside any timed step
            for blk in [self.block, self.local_block] + self.stage_blocks:
                if blk.num_nodes:
                    blk.to_csc().schedule()
        self._rev = None
        self.device_is_cuda = dev.type == "cuda"

    @property
    def num_local_rows(self):
        return self.r1 - self.r0

    def reverse_block(self):
        """Rows = padded source positions (world * width), local edges only."""
        if self._rev is None:
            self._rev = self.block.transpose()
            if self._rev.num_nodes and self.device_is_cuda:
                self._rev.to_csc().schedule()
        return self._rev

    # -- communication -----------------------------------------------------

    def _pad(self, x_local):
        if x_local.shape[0] == self.width:
            return x_local.contiguous()
        pad = torch.zeros((self.width, x_local.shape[1]), dtype=x_local.dtype,
                          device=x_local.device)
        pad[:x_local.shape[0]] = x_local
        return pad

    def all_gather(self, x_local, group=None):
        """The padded buffer holding every shard (one NCCL all-gather)."""
        import torch.distributed as dist
        out = torch.empty((self.world * self.width, x_local.shape[1]), dtype=x_local.dtype,
                          device=x_local.device)
        dist.all_gather_into_tensor(out, self._pad(x_local), group=group)
        return out

    def _shift_steps(self, x_local, gathered, steps, group=None):
        """Shift pattern: send the local shard to rank + k, receive rank - k's
        shard into its slot of the padded buffer, for every k in steps."""
        import torch.distributed as dist
        xs = x_local.contiguous()
        ops = []
        for k in steps:
            dst, src = (self.rank + k) % self.world, (self.rank - k) % self.world
            slot = gathered[src * self.width:src * self.width + self.sizes[src]]
            ops.append(dist.P2POp(dist.isend, xs, dst, group))
            ops.append(dist.P2POp(dist.irecv, slot, src, group))
        for w in dist.batch_isend_irecv(ops):
            w.wait()

    # -- forward -----------------------------------------------------------

    def aggregate(self, x_local, rho="sum", overlap=True, group=None):
        """Forward g-SpMM (copy_u sum / mean) of the local rows; x_local is
        this rank's shard. overlap=False: one all-gather, then one launch."""
        if rho not in ("sum", "mean"):
            raise ValueError("row-partitioned aggregation takes sum / mean")
        if self.world == 1:
            return stage_aggregate(self.local_block, x_local, rho)
        if not overlap:
            return stage_aggregate(self.block, self.all_gather(x_local, group), rho)
        dev = x_local.device
        d = x_local.shape[1]
        acc = torch.empty((self.num_local_rows, d), dtype=torch.float64, device=dev)
        z = torch.empty((self.num_local_rows, d), dtype=x_local.dtype, device=dev)
        deg = self.deg if rho == "mean" else None
        gathered = torch.empty((self.world * self.width, d), dtype=x_local.dtype, device=dev)
        cuda = x_local.is_cuda
        p2p = (not cuda) or _is_nccl(group)
        ready = []
        if cuda:
            compute = torch.cuda.current_stream(dev)
            comm = torch.cuda.Stream(device=dev)
            comm.wait_stream(compute)
            with torch.cuda.stream(comm):
                if p2p:
                    for steps in self.groups:
                        self._shift_steps(x_local, gathered, steps, group)
                        ready.append(comm.record_event())
                else:  # e.g. gloo on CUDA tensors: one all-gather
                    gathered.copy_(self.all_gather(x_local, group))
                    ready = [comm.record_event()] * len(self.groups)
        # stage 0 needs no communication and runs while the shards move
        stage_aggregate(self.local_block, x_local, rho, acc, STAGE_FIRST, deg, z)
        for i, blk in enumerate(self.stage_blocks):
            if cuda:
                torch.cuda.current_stream(dev).wait_event(ready[i])
            else:
                self._shift_steps(x_local, gathered, self.groups[i], group)
            last = i == len(self.stage_blocks) - 1
            stage_aggregate(blk, gathered, rho, acc, STAGE_LAST if last else STAGE_MID, deg, z)
        if cuda:
            x_local.record_stream(comm)
            gathered.record_stream(comm)
        return z

    # -- backward ----------------------------------------------------------

    def aggregate_backward(self, dz_local, rho="sum", group=None):
        """dX shard of the forward aggregation: the reverse block sums dZ (or
        dZ / deg for mean) into an fp64 full-length partial over the padded
        positions; an fp64 reduce-scatter adds the ranks' partials and each
        rank rounds its shard once."""
        import torch.distributed as dist
        dz = dz_local.contiguous()
        if rho == "mean":
            # mean backward: dZ / deg (autodiff.py:405), 0 for empty rows
            dg = self.deg.to(torch.float64).clamp_min(1).unsqueeze(1)
            dz = (dz.to(torch.float64) / dg).to(dz_local.dtype)
        rev = self.reverse_block()
        part = torch.empty((rev.num_nodes, dz.shape[1]), dtype=torch.float64, device=dz.device)
        stage_aggregate(rev, dz, "sum", part, STAGE_FIRST)
        if self.world == 1:
            return part[:self.sizes[0]].to(dz_local.dtype)
        out = torch.empty((self.width, dz.shape[1]), dtype=torch.float64, device=dz.device)
        dist.reduce_scatter_tensor(out, part, group=group)
        return out[:self.num_local_rows].to(dz_local.dtype)


class DistAggregate(torch.autograd.Function):
    """Row-partitioned copy_u + sum / mean: staged forward (local shard first,
    remote shards as they land), fp64 reduce-scatter backward."""

    @staticmethod
    def forward(ctx, x_local, pg, overlap, rho="sum"):
        ctx.pg, ctx.rho = pg, rho
        return pg.aggregate(x_local, rho, overlap=overlap)

    @staticmethod
    def backward(ctx, dz_local):
        return ctx.pg.aggregate_backward(dz_local, ctx.rho), None, None, None


class DistGCN:
    """Row-partitioned GCN (the reference's GCNModel, layers.py:137-158, on a
    PartitionedGraph): weights replicated (same seeded init on every rank),
    node rows sharded. Each layer aggregates the narrower side of W (the
    DGL GraphConv rule, layers.gcn_layer); the loss is the global mean
    cross-entropy; weight gradients are summed over ranks with one
    all-reduce of a flat buffer before the SGD update (layers.py:175-202)."""

    def __init__(self, dims, seed=0, aggregator="sum", device=None, dtype=torch.float32):
        from . import layers
        ref = layers.GCNModel(dims, seed=seed, aggregator=aggregator, device=device, dtype=dtype)
        self.layers = ref.layers
        self.aggregator = aggregator
        self.out_dim = dims[-1]

    def parameters(self):
        return [t for lp in self.layers for t in (lp.W, lp.b)]

    def forward(self, pg, x_local, overlap=True):
        from . import layers
        h = x_local
        last = len(self.layers) - 1
        for i, p in enumerate(self.layers):
            if layers._project_first(h, p.W, "auto"):
                z = DistAggregate.apply(layers._mm(h, p.W), pg, overlap, self.aggregator)
            else:
                z = layers._mm(DistAggregate.apply(h, pg, overlap, self.aggregator), p.W)
            h = z + p.b
            if i < last:
                h = torch.relu(h)
        return h

    def train_epoch(self, pg, x_local, labels_local, lr, overlap=True, group=None):
        """One full-graph gradient-descent step; returns the global loss."""
        import torch.distributed as dist
        import torch.nn.functional as F
        params = self.parameters()
        logits = self.forward(pg, x_local, overlap)
        loss_local = F.cross_entropy(logits, labels_local, reduction="sum") / pg.num_nodes
        grads = torch.autograd.grad(loss_local, params)
        flat = torch.cat([g.reshape(-1) for g in grads] + [loss_local.detach().reshape(1)])
        if pg.world > 1:
            dist.all_reduce(flat, group=group)
        with torch.no_grad():
            off = 0
            for p in params:
                k = p.numel()
                p.sub_(lr * flat[off:off + k].view_as(p))
                off += k
        return flat[-1]
