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


@pytest.fixture(params=["seg", "seg_tiny_windows", "items"])
def stats_path(request, monkeypatch):
    """seg: the chunked segmented pass over the window-major plan (default);
    seg_tiny_windows: 1024-edge windows, so pieces are a few edges long and
    most sub-steps close several pieces; items: the (window, row) work-item
    kernel (GMP_SOFTMAX_SEG=0)."""
    if request.param == "items":
        monkeypatch.setattr(kernels, "_SEG_OFF", True)
        return request.param
    monkeypatch.setattr(kernels, "_SEG_BWD_OFF", False)  # the backward's segmented pass too
    if request.param == "seg_tiny_windows":
        monkeypatch.setattr(kernels, "_SEG_WINDOW_MB", 0)
    return request.param


@pytest.mark.parametrize("shuffle", [False, True])
@pytest.mark.parametrize("H", [1, 4, 8])
def test_windowed_softmax_fwd_bwd_matches_oracle(shuffle, H, stats_path):
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


@pytest.mark.parametrize("H", [2, 8, 16])
@pytest.mark.parametrize("win_mb", [0, 40])
def test_segmented_stats_small_graph(H, win_mb, monkeypatch):
    """The segmented pass forced onto a 300k-edge graph (hub rows of 20k
    in-edges plus a uniform background, edge list shuffled): pieces of every
    length, chunk cuts inside hub segments, lane-group widths 2 / 8 / 16 for
    H = 2 / 8 / 16; fp32 and fp64 against the oracle, run-to-run identical."""
    monkeypatch.setattr(kernels, "_SEG_MIN_EDGES", 0)
    monkeypatch.setattr(kernels, "_SEG_WINDOW_MB", win_mb)
    monkeypatch.setattr(kernels, "_SEG_BWD_OFF", False)
    rng = np.random.default_rng(7)
    n, m = 30000, 300000
    d = np.where(rng.random(m) < 0.5, rng.integers(0, 8, m), rng.integers(0, n, m))
    s = rng.integers(0, n, m)
    g = G.from_arrays(s, d, num_nodes=n, device=DEV)
    assert g.to_csc().schedule().n_heavy > 0
    sc = (rng.standard_normal((m, H)) * 3).astype(np.float64)
    up = rng.standard_normal((m, H))
    want = O.edge_softmax(s, d, n, sc)
    for dt in (torch.float32, torch.float64):
        St = torch.as_tensor(sc, device=DEV).to(dt)
        alpha = kernels.edge_softmax_forward(g, St)
        ds = kernels.edge_softmax_backward(g, alpha, torch.as_tensor(up, device=DEV).to(dt))
        wds = O.edge_softmax_backward(s, d, n, to_np(alpha).astype(np.float64),
                                      to_np(torch.as_tensor(up).to(dt)).astype(np.float64))
        if dt == torch.float32:
            assert np.allclose(to_np(alpha), want, rtol=RTOL32, atol=ATOL32)
            assert np.allclose(to_np(ds), wds, rtol=RTOL32, atol=ATOL32)
        else:
            assert np.allclose(to_np(alpha), want, rtol=1e-12, atol=1e-14)
            assert np.allclose(to_np(ds), wds, rtol=1e-12, atol=1e-14)
        assert torch.equal(alpha, kernels.edge_softmax_forward(g, St))
    assert any(k[0] == "segplan" for k in g.to_csc()._extra if isinstance(k, tuple))
