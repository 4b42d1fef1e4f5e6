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


@pytest.mark.parametrize("op", ["copy", "mul", "dot", "add"])
def test_many_writer_gradients_deterministic_fp64(op):
    """Source rows (and broadcast operands) that win several cells are summed
    in fp64, in a fixed order, and rounded once (sort-grouped, no float
    atomics): fp32 gradients equal the oracle's fp64 sums rounded to fp32 to
    north_star's bar and are bit-identical run to run."""
    from oracle import gmp_oracle as O
    from conftest import assert_close32
    s, d = G.generators.power_law_edges(6000, 12, seed=7)
    n, m = 6000, s.size
    g = G.from_arrays(s, d, num_nodes=n, device=DEV)
    rng = np.random.default_rng(3)
    dd = 5
    X = rng.standard_normal((n, dd)).astype(np.float32)
    if op == "copy":
        phi, name, kw, okw = kernels.copy("src"), "copy_lhs", {}, {}
    elif op == "dot":
        Y = rng.standard_normal((n, dd)).astype(np.float32)
        phi, name = kernels.dot("src", "dst"), "dot"
        kw, okw = {"Y": torch.as_tensor(Y, device=DEV)}, {"Y": Y}
    else:
        W = rng.standard_normal((m, 1)).astype(np.float32)   # broadcast edge operand
        phi, name = kernels.MessageFunc(op, "src", "edge"), op
        kw, okw = {"W": torch.as_tensor(W, device=DEV)}, {"W": W}
    Xt = torch.as_tensor(X, device=DEV)
    z, aux = G.gspmm(g, phi, "max", X=Xt, **kw)
    dz = torch.as_tensor(rng.standard_normal(tuple(z.shape)).astype(np.float32), device=DEV)
    needs = ("x",) + tuple(k.lower() for k in kw)
    runs = [G.gspmm_backward(g, phi, "max", X=Xt, **kw, aux=aux, dZ=dz, needs=needs)
            for _ in range(3)]
    rt = None if op == "copy" else ("dst" if op == "dot" else "edge")
    want = O.gspmm_backward(s, d, n, name, "src", rt, "max",
                            X=X.astype(np.float64),
                            **{k: v.astype(np.float64) for k, v in okw.items()},
                            aux=to_np(aux.arg_edge), dZ=to_np(dz).astype(np.float64))
    for attr, key in (("dx", "src"), ("dy", "dst"), ("dw", "edge")):
        got = getattr(runs[0], attr, None)
        if got is None or key not in want:
            continue
        assert_close32(got, want[key], "%s %s" % (op, attr))
        for r in runs[1:]:
            assert torch.equal(getattr(r, attr), got), (op, attr)
