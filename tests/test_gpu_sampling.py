"""Device neighbour sampling (gmp_neighbor_sample behind neighbor_sample,
reference graph.py:218-286) and feature slicing (features.py:92-98).

* exact parity with the reference where its result is not random
  (fanout >= in-degree; tests/golden/sampling.npz, make_golden_sampling.py);
* the reference's own property tests (test_graph.py:133-190,
  test_features.py:77-105): fanout cap, zero in-degree, coverage,
  determinism, validation, subgraph soundness;
* uniformity of the k-subset draw (chi-square) and launch-shape independence.
"""

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_1909_01315_b200 as G
from conftest import to_np

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from make_golden_sampling import cases  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda"
GOLD = Path(__file__).resolve().parent / "golden" / "sampling.npz"


def g3():
    return G.from_arrays(np.array([0, 1, 2]), np.array([2, 2, 0]), num_nodes=3, device=DEV)


def test_full_fanout_matches_reference_exactly():
    gold = np.load(GOLD)
    for i, (s, d, n, seeds) in enumerate(cases()):
        g = G.from_arrays(s, d, num_nodes=n, device=DEV)
        sub = G.neighbor_sample(g, seeds.tolist(), fanout=10_000, rng_seed=i)
        su, de, _ = sub.graph.coo()
        assert np.array_equal(to_np(sub.parent_node_ids), gold["s%d/node_ids" % i]), i
        assert np.array_equal(to_np(sub.parent_edge_ids), gold["s%d/edge_ids" % i]), i
        assert np.array_equal(to_np(su), gold["s%d/sub_src" % i]), i
        assert np.array_equal(to_np(de), gold["s%d/sub_dst" % i]), i


def test_fanout_exceeds_degree():
    sub = G.neighbor_sample(g3(), [2], fanout=5, rng_seed=0)
    assert sorted(to_np(sub.parent_edge_ids).tolist()) == [0, 1]
    assert int(sub.parent_node_ids[0]) == 2
    assert sub.graph.num_edges == 2


def test_zero_in_degree():
    sub = G.neighbor_sample(g3(), [1], fanout=3, rng_seed=0)
    assert to_np(sub.parent_node_ids).tolist() == [1]
    assert sub.graph.num_edges == 0
    assert sub.graph.num_nodes == 1


def test_fanout_one_covers_both_edges():
    picked = set()
    for seed in range(40):
        sub = G.neighbor_sample(g3(), [2], fanout=1, rng_seed=seed)
        assert sub.parent_edge_ids.numel() == 1
        picked.add(int(sub.parent_edge_ids[0]))
    assert picked == {0, 1}


def test_deterministic_and_batch_independent():
    rng = np.random.default_rng(11)
    s, d = rng.integers(0, 40, 300), rng.integers(0, 40, 300)
    g = G.from_arrays(s, d, num_nodes=40, device=DEV)
    a = G.neighbor_sample(g, [0, 3, 5], fanout=2, rng_seed=9)
    b = G.neighbor_sample(g, [0, 3, 5], fanout=2, rng_seed=9)
    assert torch.equal(a.parent_edge_ids, b.parent_edge_ids)
    assert torch.equal(a.parent_node_ids, b.parent_node_ids)
    # a node's picks do not depend on which other seeds share the batch
    c = G.neighbor_sample(g, [5], fanout=2, rng_seed=9)
    ea = set(to_np(a.parent_edge_ids)[to_np(g.dst.long()[a.parent_edge_ids]) == 5].tolist())
    assert ea == set(to_np(c.parent_edge_ids).tolist())


def test_validates():
    with pytest.raises(IndexError):
        G.neighbor_sample(g3(), [5], fanout=1, rng_seed=0)
    with pytest.raises(ValueError):
        G.neighbor_sample(g3(), [0], fanout=0, rng_seed=0)


def test_subgraph_soundness():
    for seed in range(25):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(2, 31))
        m = int(rng.integers(0, 121))
        s, d = rng.integers(0, n, m), rng.integers(0, n, m)
        g = G.from_arrays(s, d, num_nodes=n, device=DEV)
        seeds = rng.integers(0, n, size=3).tolist()
        sub = G.neighbor_sample(g, seeds, fanout=3, rng_seed=seed)
        nid, eid = to_np(sub.parent_node_ids), to_np(sub.parent_edge_ids)
        ssu, sde, _ = (to_np(t) for t in sub.graph.coo())
        assert np.array_equal(nid[ssu], s[eid])
        assert np.array_equal(nid[sde], d[eid])
        assert len(set(eid.tolist())) == eid.size  # without replacement
        for v in set(seeds):
            local = int(np.flatnonzero(nid == v)[0])
            assert (sde == local).sum() == min(3, int((d == v).sum()))
        # new nodes ascending after the seeds
        k = len(dict.fromkeys(seeds))
        assert np.all(np.diff(nid[k:]) > 0)


def test_k_subsets_uniform():
    """deg 5, fanout 2: each of the 10 pairs equally likely (chi-square,
    9 dof, p = 0.001 critical value 27.9)."""
    s = np.arange(1, 6)
    g = G.from_arrays(s, np.zeros(5, dtype=np.int64), num_nodes=6, device=DEV)
    counts = {}
    trials = 4000
    for seed in range(trials):
        sub = G.neighbor_sample(g, [0], fanout=2, rng_seed=seed)
        key = tuple(to_np(sub.parent_edge_ids).tolist())
        assert list(key) == sorted(key)
        counts[key] = counts.get(key, 0) + 1
    assert len(counts) == 10
    exp = trials / 10
    chi2 = sum((c - exp) ** 2 / exp for c in counts.values())
    assert chi2 < 27.9, counts


def test_large_fanout_on_hub():
    """k in the hundreds on a 5000-edge hub row: distinct, ascending, in range."""
    s = np.random.default_rng(0).integers(1, 9000, 5000)
    g = G.from_arrays(s, np.zeros(5000, dtype=np.int64), num_nodes=9000, device=DEV)
    sub = G.neighbor_sample(g, [0], fanout=700, rng_seed=5)
    e = to_np(sub.parent_edge_ids)
    assert e.size == 700 and len(set(e.tolist())) == 700
    inv = np.empty(5000, dtype=np.int64)
    inv[to_np(g.to_csc().edge_ids)] = np.arange(5000)
    assert np.all(np.diff(inv[e]) > 0)  # ascending in-adjacency positions
    assert sub.graph.num_edges == 700


def test_slice_rows_on_subgraph():
    g = G.build_graph(3, [(0, 2), (1, 2), (2, 0)], device=DEV)
    x = torch.tensor([[10.0], [20.0], [30.0]], device=DEV)
    sub = G.neighbor_sample(g, [2], fanout=5, rng_seed=0)
    sliced = G.slice_rows(x, sub.parent_node_ids)
    assert float(sliced[0, 0]) == 30.0
    assert sorted(to_np(sliced).ravel().tolist()) == [10.0, 20.0, 30.0]
    with pytest.raises(IndexError):
        G.slice_rows(x, [3])
