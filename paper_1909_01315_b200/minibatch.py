"""Mini-batch training over sampled subgraphs (the paper's
neighbour-sampling (NS) and cluster-sampling (CS) benchmarks).

The reference ships the single-hop sampler (neighbor_sample / Subgraph,
/root/reference/pkg/src/graphmp/graph.py:218-286) and slice_rows
(features.py:92-98); the multi-layer block construction and the two epoch
loops here are built on exactly those pieces, on the device:

* ns_blocks: for an L-layer model with fanouts [f_0 .. f_{L-1}] (f_0 for the
  input layer), the output seeds are sampled with f_{L-1}; the nodes of that
  block become the seeds of the block below, and so on. A block's seeds come
  first in its relabelling (graph.py:238-240), so the rows a layer must
  produce for the next block are exactly its first rows - no index remap
  between layers;
* node_subgraph: the subgraph induced by a node set (Cluster-GCN style CS),
  nodes relabelled in the given order, edges kept in parent edge-id order;
* train_ns_epoch / train_cs_epoch: one pass over the training seeds / the
  clusters, one SGD step per batch through the same kernels as full-graph
  training (the blocks are ordinary Graphs, so every g-SpMM, its reverse-graph
  backward and the fused GAT path run unchanged).
"""

import numpy as np
import torch

from .features import slice_rows
from .graph import Graph, Subgraph, neighbor_sample
from .layers import xent_loss


def ns_blocks(g, seeds, fanouts, rng_seed):
    """Blocks for a len(fanouts)-layer model, input layer first."""
    if not fanouts:
        raise ValueError("need one fanout per layer")
    blocks = []
    cur = seeds
    for i, f in enumerate(reversed(list(fanouts))):
        sub = neighbor_sample(g, cur, int(f), (int(rng_seed) * 1000003 + i) & (2 ** 63 - 1))
        blocks.append(sub)
        cur = sub.parent_node_ids
    return blocks[::-1]


def forward_blocks(model, blocks, x_in):
    """Run layer i of `model` on blocks[i]; each layer keeps the rows that are
    the next block's nodes (its first rows), the last keeps the seeds."""
    h = x_in
    for i, b in enumerate(blocks):
        h = model.layer(i, b.graph, h)
        keep = blocks[i + 1].graph.num_nodes if i + 1 < len(blocks) else None
        if keep is not None:
            h = h[:keep]
    return h


def node_subgraph(g, nodes):
    """Subgraph induced by `nodes` (distinct ids): node i = nodes[i], edges
    with both endpoints inside, in parent edge-id order."""
    dev = g.device
    nodes = torch.as_tensor(nodes, dtype=torch.int64, device=dev).reshape(-1)
    relabel = torch.full((g.num_nodes,), -1, dtype=torch.int64, device=dev)
    relabel[nodes] = torch.arange(nodes.numel(), dtype=torch.int64, device=dev)
    rs = relabel.index_select(0, g.src.to(torch.int64))
    rd = relabel.index_select(0, g.dst.to(torch.int64))
    keep = torch.nonzero((rs >= 0) & (rd >= 0)).reshape(-1)
    sub = Graph(rs.index_select(0, keep), rd.index_select(0, keep), nodes.numel(), device=dev)
    return Subgraph(sub, nodes, keep)


def _sgd(loss, params, lr):
    grads = torch.autograd.grad(loss, params)
    with torch.no_grad():
        for p, gr in zip(params, grads):
            p.sub_(lr * gr)


def train_ns_epoch(g, x, labels, model, lr, train_nodes, batch_size, fanouts, seed=0):
    """One NS epoch: shuffled training seeds in batches, per batch blocks ->
    forward -> cross-entropy on the seeds -> SGD. Returns the mean loss
    (a device tensor) and the batch count."""
    train_nodes = torch.as_tensor(train_nodes, dtype=torch.int64, device=g.device)
    gen = torch.Generator(device="cpu")
    gen.manual_seed(int(seed))
    perm = train_nodes[torch.randperm(train_nodes.numel(), generator=gen).to(g.device)]
    params = model.parameters()
    total = torch.zeros((), dtype=torch.float64, device=g.device)
    nb = 0
    for b0 in range(0, perm.numel(), batch_size):
        seeds = perm[b0:b0 + batch_size]
        blocks = ns_blocks(g, seeds, fanouts, seed * 7919 + nb)
        h = forward_blocks(model, blocks, slice_rows(x, blocks[0].parent_node_ids))
        loss = xent_loss(h[:seeds.numel()], labels.index_select(0, seeds))
        _sgd(loss, params, lr)
        total += loss.detach()
        nb += 1
    return total / max(nb, 1), nb


def cluster_partition(num_nodes, num_clusters):
    """Contiguous node-id ranges (a locality-preserving stand-in for METIS:
    the generators number nodes in attachment order)."""
    bounds = np.linspace(0, num_nodes, num_clusters + 1).astype(np.int64)
    return [(int(a), int(b)) for a, b in zip(bounds, bounds[1:]) if b > a]


def train_cs_epoch(g, x, labels, model, lr, clusters, clusters_per_batch, train_mask=None,
                   seed=0):
    """One CS (Cluster-GCN) epoch: the clusters in a shuffled order, each batch
    the subgraph induced by `clusters_per_batch` of them, full-graph forward on
    it, loss on its training nodes."""
    rng = np.random.default_rng(seed)
    order = rng.permutation(len(clusters))
    params = model.parameters()
    total = torch.zeros((), dtype=torch.float64, device=g.device)
    nb = 0
    for b0 in range(0, len(order), clusters_per_batch):
        ids = torch.cat([torch.arange(*clusters[c], device=g.device)
                         for c in order[b0:b0 + clusters_per_batch]])
        sub = node_subgraph(g, ids)
        h = model.forward(sub.graph, slice_rows(x, ids))
        lab = labels.index_select(0, ids)
        if train_mask is not None:
            sel = torch.nonzero(train_mask.index_select(0, ids)).reshape(-1)
            h, lab = h.index_select(0, sel), lab.index_select(0, sel)
        loss = xent_loss(h, lab)
        _sgd(loss, params, lr)
        total += loss.detach()
        nb += 1
    return total / max(nb, 1), nb
