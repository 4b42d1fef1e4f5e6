"""fp32 edge_softmax and fused GAT attention at large score magnitudes.

The reference's softmax is "always max-stabilised" (
messaging.py:105-126), and its tests shift scores and feed +-1000 extremes
(test_messaging.py:130-143). In fp32 a softmax exponent formed as
x*log2e - m*log2e carries an error proportional to |m|, which stops
cancelling once partials with different maxima are merged (online rescale,
slot / warp / window / cluster merges). These tests pin the fix: every fp32
term is exp((x - m)) with the error relative to |x - m| (and u_add_v scores
carried as an exact pair), so results meet rtol 1e-5 / atol 1e-6 elementwise
at any offset. Graphs: a hub graph (a 5000-edge row on the CTA path, rows
split over lane slots and warps) and the 4.8M-edge graph that takes the
windowed statistics path."""

import numpy as np
import pytest
import torch

import paper_1909_01315_b200 as G
from paper_1909_01315_b200 import autodiff, kernels
from oracle import gmp_oracle as O
from conftest import assert_close32, to_np

pytestmark = pytest.mark.gpu
DEV = "cuda"


def hub_graph(n=6000, seed=0):
    rng = np.random.default_rng(seed)
    s, d = G.generators.power_law_edges(n, 8, seed=seed)
    extra = rng.integers(0, n - 50, 5000)
    return np.concatenate([s, extra]), np.concatenate([d, np.full(5000, 7)]), n


def window_graph():
    s, d = G.generators.power_law_edges(60000, 80, seed=4)
    return s, d, 60000


_GRAPHS = {}


def graph(kind):
    if kind not in _GRAPHS:
        s, d, n = hub_graph() if kind == "hub" else window_graph()
        _GRAPHS[kind] = (s, d, n, G.from_arrays(s, d, num_nodes=n, device=DEV))
    return _GRAPHS[kind]


def shifted_scores(m, H, d, offset, seed):
    """N(0,1) scores + offset; offset 'mixed' gives rows alternately +1000 and
    -1000 (by destination parity) and a few in-row +-1000 extremes."""
    rng = np.random.default_rng(seed)
    sc = rng.standard_normal((m, H))
    if offset == "mixed":
        sc += np.where(d % 2 == 0, 1000.0, -1000.0)[:, None]
        ext = rng.choice(m, size=max(1, m // 1000), replace=False)
        sc[ext] += rng.choice([-1000.0, 1000.0], size=(ext.size, 1))
    else:
        sc += float(offset)
    return sc.astype(np.float32)


@pytest.mark.parametrize("H", [1, 8])
@pytest.mark.parametrize("offset", [0, 300, 1000, 3000, -1000, "mixed"])
def test_softmax_offsets_hub_graph(H, offset):
    s, d, n, g = graph("hub")
    sc = shifted_scores(s.size, H, d, offset, seed=H)
    up = np.random.default_rng(9).standard_normal((s.size, H)).astype(np.float32)
    alpha = kernels.edge_softmax_forward(g, torch.as_tensor(sc, device=DEV))
    want = O.edge_softmax(s, d, n, sc.astype(np.float64))
    assert_close32(alpha, want, "alpha H=%d offset=%s" % (H, offset))
    ds = kernels.edge_softmax_backward(g, alpha, torch.as_tensor(up, device=DEV))
    wds = O.edge_softmax_backward(s, d, n, to_np(alpha).astype(np.float64), up.astype(np.float64))
    assert_close32(ds, wds, "ds H=%d offset=%s" % (H, offset))


@pytest.mark.parametrize("H", [1, 8])
@pytest.mark.parametrize("offset", [1000, 3000, "mixed"])
def test_softmax_offsets_windowed(H, offset):
    s, d, n, g = graph("window")
    assert g.to_csc().schedule().n_heavy > 0 and s.size >= (1 << 22)
    sc = shifted_scores(s.size, H, d, offset, seed=10 + H)
    up = np.random.default_rng(11).standard_normal((s.size, H)).astype(np.float32)
    alpha = kernels.edge_softmax_forward(g, torch.as_tensor(sc, device=DEV))
    want = O.edge_softmax(s, d, n, sc.astype(np.float64))
    assert_close32(alpha, want, "alpha windowed H=%d offset=%s" % (H, offset))
    ds = kernels.edge_softmax_backward(g, alpha, torch.as_tensor(up, device=DEV))
    wds = O.edge_softmax_backward(s, d, n, to_np(alpha).astype(np.float64), up.astype(np.float64))
    assert_close32(ds, wds, "ds windowed H=%d offset=%s" % (H, offset))


def test_softmax_uv_large_scores():
    """Fused u_add_v + edge_softmax: el ~ +600, er ~ +-400, so the fp32 sum
    el + er is not exact - the exact pair keeps alpha at parity."""
    s, d, n, g = graph("hub")
    rng = np.random.default_rng(2)
    for H in (1, 8):
        el = (rng.standard_normal((n, H)) * 3 + 600).astype(np.float32)
        er = (rng.standard_normal((n, H)) * 3 + np.where(np.arange(n) % 2, 400, -400)[:, None]
              ).astype(np.float32)
        alpha = kernels.edge_softmax_uv_forward(g, torch.as_tensor(el, device=DEV),
                                                torch.as_tensor(er, device=DEV))
        sc = el.astype(np.float64)[s] + er.astype(np.float64)[d]
        assert_close32(alpha, O.edge_softmax(s, d, n, sc), "uv alpha H=%d" % H)


@pytest.mark.parametrize("shared,H,dh", [(False, 1, 16), (False, 4, 8), (True, 2, 5)])
@pytest.mark.parametrize("offset", [1000, 3000])
def test_fused_gat_large_scores(shared, H, dh, offset):
    from test_gpu_gat_fused import oracle_gat, oracle_grads
    s, d, n, g = graph("hub")
    rng = np.random.default_rng(H * 10 + dh)
    el = (rng.standard_normal((n, H)) + offset * 0.5).astype(np.float32)
    er = (rng.standard_normal((n, H)) + offset * 0.5).astype(np.float32)
    X = rng.standard_normal((n, dh if shared else H * dh)).astype(np.float32)
    dout = rng.standard_normal((n, H * dh)).astype(np.float32)
    t = [torch.as_tensor(a, device=DEV).requires_grad_(True) for a in (el, er, X)]
    out = autodiff.gat_attention(g, t[0], t[1], t[2], shared=shared)
    (out * torch.as_tensor(dout, device=DEV)).sum().backward()
    f64 = lambda a: a.astype(np.float64)  # noqa: E731
    want, _ = oracle_gat(s, d, n, f64(el), f64(er), f64(X), shared)
    wdX, wdEl, _ = oracle_grads(s, d, n, f64(el), f64(er), f64(X), shared, f64(dout))
    assert_close32(out, want, "gat out")
    assert_close32(t[2].grad, wdX, "gat dX")
    assert_close32(t[0].grad, wdEl, "gat d el")
    assert float(t[1].grad.abs().max()) == 0.0
