"""Messaging API, autograd and layers on the GPU path (reference semantics)."""

import numpy as np
import pytest
import torch

import paper_1909_01315_b200 as G
from paper_1909_01315_b200 import kernels, layers
from conftest import assert_close32, golden, golden_graph, rel_err, to_np

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _g3_stores(dtype=torch.float64):
    g = G.build_graph(3, [(0, 2), (1, 2), (2, 0)], device=DEV)
    nd, ed = G.FeatureDict(3), G.FeatureDict(3)
    nd["h"] = torch.tensor([[1.0], [2.0], [3.0]], dtype=dtype, device=DEV)
    ed["w"] = torch.tensor([[10.0], [20.0], [30.0]], dtype=dtype, device=DEV)
    return g, nd, ed


def test_update_all_and_apply_edges_frozen():
    g, nd, ed = _g3_stores()
    z = G.update_all(g, G.msg("copy", G.src("h")), "sum", nd, out="z")
    assert z.tolist() == [[3.0], [0.0], [3.0]] and torch.equal(nd.array("z"), z)
    z = G.update_all(g, G.msg("mul", G.src("h"), G.edge("w")), "sum", nd, ed, out="z")
    assert z.tolist() == [[90.0], [0.0], [50.0]]
    nd["p"] = torch.tensor([[1.0, 0.0], [0.0, 1.0], [1.0, 1.0]], device=DEV)
    m = G.apply_edges(g, G.msg("dot", G.src("p"), G.dst("p")), nd, ed, out="s")
    assert m.tolist() == [[1.0], [1.0], [1.0]] and "s" in ed
    with G.capture_dispatch() as log:
        G.update_all(g, G.msg("mul", G.src("h"), G.edge("w")), "sum", nd, ed, out="z")
        G.apply_edges(g, G.msg("sub", G.dst("h"), G.src("h")), nd, ed, out="d")
        G.edge_softmax(g, "w", ed, out="a")
    assert [r.kernel for r in log] == ["gspmm", "gsddmm", "gspmm"]  # softmax: ONE fused launch
    assert "a" in ed


def test_two_hop_matches_dense_power():
    rng = np.random.default_rng(0)
    n, m = 20, 60
    s, d = rng.integers(0, n, m), rng.integers(0, n, m)
    g = G.from_arrays(s, d, n, device=DEV)
    x = rng.standard_normal((n, 3))
    a = np.zeros((n, n))
    np.add.at(a, (s, d), 1.0)
    nd = G.FeatureDict(n)
    nd["h"] = x
    G.update_all(g, G.msg("copy", G.src("h")), "sum", nd, out="h1")
    G.update_all(g, G.msg("copy", G.src("h1")), "sum", nd, out="h2")
    assert rel_err(to_np(nd.array("h2")), a.T @ a.T @ x) < 1e-12


def test_edge_softmax_properties():
    rng = np.random.default_rng(2)
    for _ in range(5):
        n, m = 30, 120
        s, d = rng.integers(0, n, m), rng.integers(0, n, m)
        g = G.from_arrays(s, d, n, device=DEV)
        sc = torch.as_tensor(rng.standard_normal((m, 3)) * 50, device=DEV)
        alpha = G.edge_softmax(g, sc)
        sums, _ = G.gspmm(g, kernels.copy_rhs("edge"), "sum", W=alpha)
        cnt = to_np(g.in_degrees())
        assert np.allclose(to_np(sums)[cnt > 0], 1.0, atol=1e-12)
        assert not to_np(sums)[cnt == 0].any()
        a1 = G.edge_softmax(g, sc + 7.25)
        assert rel_err(to_np(a1), to_np(alpha)) < 1e-12
    g = G.build_graph(2, [(0, 1), (1, 1)], device=DEV)
    alpha = G.edge_softmax(g, np.array([[1000.0], [-1000.0]]))
    assert bool(torch.isfinite(alpha).all()) and abs(float(alpha[0, 0]) - 1.0) < 1e-12


def test_backward_runs_on_reverse_graph():
    g = G.build_graph(3, [(0, 2), (1, 2), (2, 0)], device=DEV)
    rev = G.reverse(g)
    x = torch.tensor([[1.0], [2.0], [3.0]], dtype=torch.float64, device=DEV)
    g.to_csc(), g.to_csr()
    n_before = g.adjacency_build_count
    with G.capture_dispatch() as log:
        G.gspmm_backward(g, kernels.copy("src"), "sum", X=x, dZ=torch.ones_like(x), needs=("x",))
    spmm = [r.graph_id for r in log if r.kernel == "gspmm"]
    assert rev.uid in spmm and g.uid not in spmm
    assert g.adjacency_build_count == n_before
    b = G.gspmm_backward(g, kernels.mul("src", "edge"), "sum", X=x,
                         W=torch.tensor([[10.0], [20.0], [30.0]], dtype=torch.float64, device=DEV),
                         dZ=torch.ones_like(x))
    assert b.dw.tolist() == [[1.0], [2.0], [3.0]] and b.dx.tolist() == [[10.0], [20.0], [30.0]]


def test_extrema_backward_routes_only_arg_edge():
    g = G.build_graph(3, [(0, 2), (1, 2)], device=DEV)
    x = torch.tensor([[1.0], [5.0], [0.0]], dtype=torch.float64, device=DEV)
    z, aux = G.gspmm(g, kernels.copy("src"), "max", X=x)
    b = G.gspmm_backward(g, kernels.copy("src"), "max", X=x, aux=aux,
                         dZ=torch.tensor([[0.0], [0.0], [9.0]], dtype=torch.float64, device=DEV))
    assert b.dx.tolist() == [[0.0], [9.0], [0.0]]
    w = torch.tensor([[1.0], [5.0]], dtype=torch.float64, device=DEV)
    zw, auxw = G.gspmm(g, kernels.copy_rhs("edge"), "max", W=w)
    bw = G.gspmm_backward(g, kernels.copy_rhs("edge"), "max", W=w, aux=auxw,
                          dZ=torch.tensor([[0.0], [0.0], [9.0]], dtype=torch.float64, device=DEV))
    assert bw.dw.tolist() == [[0.0], [9.0]]


def test_autograd_matches_gradcheck_fp64():
    rng = np.random.default_rng(5)
    n, m = 10, 30
    s, d = rng.integers(0, n, m), rng.integers(0, n, m)
    g = G.from_arrays(s, d, n, device=DEV)
    for phi, shapes in ((kernels.mul("src", "edge"), {"X": (n, 2), "W": (m, 1)}),
                        (kernels.add("src", "dst"), {"X": (n, 3), "Y": (n, 3)}),
                        (kernels.div("edge", "dst"), {"W": (m, 2), "Y": (n, 2)}),
                        (kernels.dot("src", "edge"), {"X": (n, 4), "W": (m, 4)})):
        ops = {k: torch.as_tensor(np.abs(rng.standard_normal(v)) + 0.5, device=DEV)
               .requires_grad_(True) for k, v in shapes.items()}
        names = sorted(ops)

        def f(*args):
            kw = dict(zip(names, args))
            z = G.autodiff.gspmm(g, phi, "sum", **kw)
            e = G.autodiff.gsddmm(g, phi, **kw)
            return z.sum() + (e * e).sum()

        assert torch.autograd.gradcheck(f, tuple(ops[k] for k in names), eps=1e-6, atol=1e-6)
    sc = torch.as_tensor(rng.standard_normal((m, 2)), device=DEV).requires_grad_(True)
    assert torch.autograd.gradcheck(lambda t: (G.edge_softmax(g, t) ** 2).sum(), (sc,),
                                    eps=1e-6, atol=1e-6)


@pytest.mark.parametrize("order", ["auto", "aggregate_first", "project_first"])
def test_gcn_training_losses_match_reference(order):
    gd = golden()
    src, dst, n = golden_graph("gcn")
    g = G.from_arrays(src.astype(np.int64), dst.astype(np.int64), n, device=DEV)
    want = gd["gcn/losses"]
    model = layers.GCNModel([12, 8, 3], seed=0, dtype=torch.float64, order=order)
    losses = layers.train(g, gd["gcn/x"].astype(np.float64), gd["gcn/labels"], model,
                          layers.TrainConfig(lr=0.1, epochs=5))
    assert np.allclose(losses, want, rtol=1e-10, atol=1e-12)
    model32 = layers.GCNModel([12, 8, 3], seed=0, dtype=torch.float32, order=order)
    l32 = layers.train(g, gd["gcn/x"], gd["gcn/labels"], model32,
                       layers.TrainConfig(lr=0.1, epochs=5))
    assert np.allclose(l32, want, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("fused", [True, False])
def test_gat_layer_matches_reference(fused):
    gd = golden()
    src, dst, n = golden_graph("gcn")
    g = G.from_arrays(src.astype(np.int64), dst.astype(np.int64), n, device=DEV)
    params = layers.init_gat(np.random.default_rng(1), 12, 4, 3)
    h = layers.gat_layer(g, torch.as_tensor(gd["gcn/x"].astype(np.float64), device=DEV), params,
                         fused=fused)
    assert rel_err(to_np(h), gd["gat/out"]) < 1e-10


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_fused_uv_softmax_matches_composition(dtype):
    """edge_softmax(u_add_v(el, er)) fused vs gsddmm(add) then edge_softmax.
    The fused kernels carry the score el + er as an exact pair, so they match
    the oracle on the exact scores; the composition matches it on the
    fp32-rounded scores it stores. Both within north_star's fp32 bar, the
    gradients too."""
    from oracle import gmp_oracle as O
    s, d = G.generators.power_law_edges(5000, 10, seed=2)
    g = G.from_arrays(s, d, num_nodes=5000, device=DEV)
    for H in (1, 3, 8):
        el = torch.randn(5000, H, device=DEV, dtype=dtype).requires_grad_(True)
        er = torch.randn(5000, H, device=DEV, dtype=dtype).requires_grad_(True)
        u = torch.randn(g.num_edges, H, device=DEV, dtype=dtype)
        a1 = G.autodiff.edge_softmax_uv(g, el, er)
        (a1 * u).sum().backward()
        g1 = (el.grad.clone(), er.grad.clone())
        el.grad = er.grad = None
        score = G.autodiff.gsddmm(g, kernels.add("src", "dst"), X=el, Y=er)
        a2 = G.edge_softmax(g, score)
        (a2 * u).sum().backward()
        exact = to_np(el).astype(np.float64)[s] + to_np(er).astype(np.float64)[d]
        want1 = O.edge_softmax(s, d, 5000, exact)
        want2 = O.edge_softmax(s, d, 5000, to_np(score).astype(np.float64))
        if dtype == torch.float64:
            assert rel_err(to_np(a1), want1) < 1e-12 and rel_err(to_np(a2), want2) < 1e-12
            assert rel_err(to_np(g1[0]), to_np(el.grad)) < 1e-12
            assert rel_err(to_np(g1[1]), to_np(er.grad)) < 1e-12
        else:
            assert_close32(a1, want1, "fused alpha H=%d" % H)
            assert_close32(a2, want2, "composed alpha H=%d" % H)
            assert_close32(g1[0], to_np(el.grad).astype(np.float64), "d el H=%d" % H)
            assert_close32(g1[1], to_np(er.grad).astype(np.float64), "d er H=%d" % H)


def test_host_pipeline_matches_device_gspmm():
    from paper_1909_01315_b200 import pipeline
    s, d = G.generators.power_law_edges(20000, 30, seed=4)
    g = G.from_arrays(s, d, num_nodes=20000, device=DEV)
    for F in (62, 130, 602):
        x = torch.randn(20000, F, dtype=torch.float32).pin_memory()
        z = torch.empty(20000, F, dtype=torch.float32).pin_memory()
        for rho in ("sum", "mean"):
            pipeline.gspmm_host(g, x, z, rho)
            torch.cuda.synchronize()
            want, _ = G.gspmm(g, kernels.copy("src"), rho, X=x.to(DEV))
            assert torch.equal(z, want.cpu()), (F, rho)
