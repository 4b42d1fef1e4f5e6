"""Fused max/min backward of binary messages (gmp_extrema_bwd_binary)
against the composed path it replaces (route_extrema_grad's dense (m, d)
matrix, then the Theorem-1 edge gradients, autodiff.py:289-412) on a
power-law graph with hub rows: destination / edge gradients of full-width
operands bit-exact, source rows and broadcast operands within tolerance."""

import numpy as np
import pytest
import torch

import paper_1909_01315_b200 as G
from paper_1909_01315_b200 import autodiff, kernels
from conftest import to_np

pytestmark = pytest.mark.gpu
DEV = "cuda"

PAIRS = [("src", "dst"), ("dst", "src"), ("src", "edge"), ("edge", "src"), ("dst", "edge"),
         ("edge", "dst")]


@pytest.mark.parametrize("op", ["add", "sub", "mul", "div", "dot"])
@pytest.mark.parametrize("rho", ["max", "min"])
@pytest.mark.parametrize("bcast", [False, True])
def test_fused_binary_extrema_backward_matches_composition(op, rho, bcast):
    if op == "dot" and bcast:
        pytest.skip("dot needs equal operand widths (kernels.py:242-246)")
    s, d = G.generators.power_law_edges(4000, 10, seed=5)
    n, m = 4000, s.size
    g = G.from_arrays(s, d, num_nodes=n, device=DEV)
    rng = np.random.default_rng(11)
    dd = 6
    for lt, rt in PAIRS:
        phi = kernels.MessageFunc(op, lt, rt)
        dims = {lt: dd, rt: 1 if bcast else dd}
        rows = {"src": n, "dst": n, "edge": m}
        slot = {"src": "X", "dst": "Y", "edge": "W"}
        ops = {}
        for t in (lt, rt):
            a = rng.standard_normal((rows[t], dims[t]))
            if op == "div":
                a = np.abs(a) + 0.5
            ops[slot[t]] = torch.as_tensor(a, dtype=torch.float64, device=DEV)
        z, aux = G.gspmm(g, phi, rho, **ops)
        dz = torch.as_tensor(rng.standard_normal(tuple(z.shape)), device=DEV)
        needs = tuple(k.lower() for k in ops)
        fused = G.gspmm_backward(g, phi, rho, **ops, aux=aux, dZ=dz, needs=needs)
        up = kernels.route_extrema_grad(g, aux, dz, dz.shape[1])
        comp = autodiff._edge_grads(g, phi, ops.get("X"), ops.get("Y"), ops.get("W"), up,
                                    "edge", needs)
        for t in (lt, rt):
            attr = {"src": "dx", "dst": "dy", "edge": "dw"}[t]
            got, want = to_np(getattr(fused, attr)), to_np(getattr(comp, attr))
            if t != "src" and dims[t] == dd:
                assert np.array_equal(got, want), (op, rho, lt, rt, t)
            else:
                assert np.allclose(got, want, rtol=1e-12, atol=1e-12), (op, rho, lt, rt, t)


def test_fused_binary_extrema_logs_no_dense_route():
    s, d = G.generators.power_law_edges(500, 5, seed=1)
    g = G.from_arrays(s, d, num_nodes=500, device=DEV)
    X = torch.randn((500, 4), device=DEV, dtype=torch.float64)
    W = torch.randn((s.size, 1), device=DEV, dtype=torch.float64)
    z, aux = G.gspmm(g, kernels.mul("src", "edge"), "max", X=X, W=W)
    with G.capture_dispatch() as log:
        G.gspmm_backward(g, kernels.mul("src", "edge"), "max", X=X, W=W, aux=aux,
                         dZ=torch.ones_like(z), needs=("x", "w"))
    assert [r.phi for r in log] == ["argext_grad(mul(src,edge),0)", "argext_grad(mul(src,edge),1)"]
