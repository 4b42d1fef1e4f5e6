"""Windowed edge_softmax statistics (heavy rows walked in L2-sized edge-id
windows, partials merged in window order) against the oracle, on graphs
large enough to take that path (>= 4M edges, rows > 2048 in-edges), with the
edge list grouped by source (edge ids ascend inside CSC rows) and shuffled
(a per-row sorted copy of the edge ids is built)."""

import numpy as np
import pytest
import torch

import paper_1909_01315_b200 as G
from paper_1909_01315_b200 import kernels
from oracle import gmp_oracle as O
from conftest import ATOL32, RTOL32, to_np

pytestmark = pytest.mark.gpu
DEV = "cuda"


def big_graph(shuffle):
    s, d = G.generators.power_law_edges(60000, 80, seed=4)
    if shuffle:
        p = np.random.default_rng(0).permutation(s.size)
        s, d = s[p], d[p]
    return s, d, 60000


@pytest.mark.parametrize("shuffle", [False, True])
@pytest.mark.parametrize("H", [1, 4, 8])
def test_windowed_softmax_fwd_bwd_matches_oracle(shuffle, H):
    s, d, n = big_graph(shuffle)
    assert s.size >= (1 << 22)
    g = G.from_arrays(s, d, num_nodes=n, device=DEV)
    assert g.to_csc().schedule().n_heavy > 0
    rng = np.random.default_rng(H)
    sc = rng.standard_normal((s.size, H)).astype(np.float32)
    up = rng.standard_normal((s.size, H)).astype(np.float32)
    St = torch.as_tensor(sc, device=DEV)
    alpha = kernels.edge_softmax_forward(g, St)
    ds = kernels.edge_softmax_backward(g, alpha, torch.as_tensor(up, device=DEV))
    assert kernels._sorted_eids(g.to_csc()) is not None
    want = O.edge_softmax(s, d, n, sc.astype(np.float64))
    assert np.allclose(to_np(alpha), want, rtol=RTOL32, atol=ATOL32)
    wds = O.edge_softmax_backward(s, d, n, to_np(alpha).astype(np.float64), up.astype(np.float64))
    assert np.allclose(to_np(ds), wds, rtol=RTOL32, atol=ATOL32)
    # deterministic run to run
    assert torch.equal(alpha, kernels.edge_softmax_forward(g, St))


def test_windowed_sorted_eids_cache():
    s, d, n = big_graph(False)
    g = G.from_arrays(s, d, num_nodes=n, device=DEV)
    adj = g.to_csc()
    assert kernels._sorted_eids(adj) is adj.edge_ids  # already ascending inside rows
    s2, d2, _ = big_graph(True)
    g2 = G.from_arrays(s2, d2, num_nodes=n, device=DEV)
    a2 = g2.to_csc()
    se = kernels._sorted_eids(a2)
    assert se is not a2.edge_ids
    ip = to_np(a2.indptr)
    se_np, e_np = to_np(se), to_np(a2.edge_ids)
    for r in np.flatnonzero(np.diff(ip) > 2048)[:5]:
        seg = se_np[ip[r]:ip[r + 1]]
        assert np.all(np.diff(seg) > 0)
        assert np.array_equal(np.sort(e_np[ip[r]:ip[r + 1]]), seg)
