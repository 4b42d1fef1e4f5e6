"""Mini-batch path: multi-layer NS blocks, induced
subgraphs for cluster sampling, and the NS / CS epoch loops.

With every fanout >= the maximum in-degree the sampled blocks contain every
in-edge of every node a seed depends on, so a block forward must equal the
full-graph forward on the seed rows (the reference's sampler is exact in that
regime too, tests/golden/sampling.npz)."""

import numpy as np
import pytest
import torch

import paper_1909_01315_b200 as G
from paper_1909_01315_b200 import layers, minibatch
from conftest import assert_close32, to_np

pytestmark = pytest.mark.gpu
DEV = "cuda"


def graph(n=3000, deg=8, seed=3):
    s, d = G.generators.power_law_edges(n, deg, seed=seed)
    return G.from_arrays(s, d, num_nodes=n, device=DEV), s, d, n


@pytest.mark.parametrize("kind", ["sage", "gcn", "gat"])
def test_full_fanout_blocks_equal_full_graph(kind):
    g, s, d, n = graph()
    maxdeg = int(to_np(g.in_degrees()).max())
    rng = np.random.default_rng(0)
    x = torch.as_tensor(rng.standard_normal((n, 24)).astype(np.float32), device=DEV)
    if kind == "sage":
        model = layers.SAGEModel([24, 16, 5], seed=1, device=DEV)
    elif kind == "gcn":
        model = layers.GCNModel([24, 16, 5], seed=1, device=DEV)
    else:
        model = layers.GATModel([24, 16, 5], heads=2, seed=1, device=DEV)
    seeds = torch.as_tensor(rng.choice(n, 200, replace=False), device=DEV)
    blocks = minibatch.ns_blocks(g, seeds, [maxdeg, maxdeg], rng_seed=5)
    assert torch.equal(blocks[-1].parent_node_ids[:200], seeds)
    # a block's seeds are the first nodes of the block below
    k = blocks[1].graph.num_nodes
    assert torch.equal(blocks[0].parent_node_ids[:k], blocks[1].parent_node_ids)
    with torch.no_grad():
        got = minibatch.forward_blocks(model, blocks, x[blocks[0].parent_node_ids])[:200]
        want = model.forward(g, x)[seeds]
    assert_close32(got, to_np(want), "%s block forward" % kind)


def test_fanout_caps_block_in_degree():
    g, s, d, n = graph()
    seeds = torch.arange(0, n, 7, device=DEV)
    blocks = minibatch.ns_blocks(g, seeds, [3, 2], rng_seed=1)
    for b, f in zip(blocks, [3, 2]):
        deg = to_np(b.graph.in_degrees())
        assert deg.max() <= f
        # every sampled edge is a parent edge between the mapped endpoints
        pe = to_np(b.parent_edge_ids)
        ids = to_np(b.parent_node_ids)
        assert np.array_equal(ids[to_np(b.graph.src)], s[pe])
        assert np.array_equal(ids[to_np(b.graph.dst)], d[pe])


def test_node_subgraph_matches_numpy():
    g, s, d, n = graph()
    rng = np.random.default_rng(2)
    nodes = rng.choice(n, 900, replace=False)
    sub = minibatch.node_subgraph(g, nodes)
    inv = np.full(n, -1)
    inv[nodes] = np.arange(nodes.size)
    keep = np.nonzero((inv[s] >= 0) & (inv[d] >= 0))[0]
    assert np.array_equal(to_np(sub.parent_edge_ids), keep)
    assert np.array_equal(to_np(sub.graph.src), inv[s[keep]])
    assert np.array_equal(to_np(sub.graph.dst), inv[d[keep]])
    assert sub.graph.num_nodes == nodes.size


def test_ns_and_cs_epochs_learn():
    g, s, d, n = graph(n=4000, deg=10)
    rng = np.random.default_rng(4)
    x = torch.as_tensor(rng.standard_normal((n, 32)).astype(np.float32), device=DEV)
    labels = torch.as_tensor((to_np(x)[:, :4].sum(1) > 0).astype(np.int64), device=DEV)
    model = layers.SAGEModel([32, 16, 2], seed=0, device=DEV)
    train = torch.arange(0, n, device=DEV)
    losses = [float(minibatch.train_ns_epoch(g, x, labels, model, 0.5, train, 512, [10, 5],
                                             seed=e)[0]) for e in range(4)]
    assert losses[-1] < losses[0], losses
    # the labels are a function of a node's own features: SAGE keeps a self
    # term, the reference's mean GCN (no self loop) cannot see them
    model2 = layers.SAGEModel([32, 16, 2], seed=0, device=DEV)
    parts = minibatch.cluster_partition(n, 16)
    cl = [float(minibatch.train_cs_epoch(g, x, labels, model2, 0.5, parts, 4, seed=e)[0])
          for e in range(4)]
    assert cl[-1] < cl[0], cl
