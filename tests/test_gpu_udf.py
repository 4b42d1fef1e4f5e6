"""Degree-bucketed UDF path (update_all_udf, reference messaging.py:137-185)
on the device, following the reference's own UDF tests
(test_messaging.py:188-272, test_acceptance.py:243-290) with torch reducers:
results against the oracle's g-SpMM, bucket order and shapes, the size guard
and the shape errors."""

import warnings

import numpy as np
import pytest
import torch

import paper_1909_01315_b200 as G
from paper_1909_01315_b200 import kernels
from oracle import gmp_oracle as O
from conftest import rel_err, to_np

pytestmark = pytest.mark.gpu
DEV = "cuda"

REDUCERS = {"sum": lambda b: b.sum(dim=1), "mean": lambda b: b.mean(dim=1),
            "max": lambda b: b.amax(dim=1), "min": lambda b: b.amin(dim=1)}


def random_graph(rng, max_nodes, max_edges, min_nodes=1):
    n = int(rng.integers(min_nodes, max_nodes + 1))
    m = int(rng.integers(0, max_edges + 1))
    return rng.integers(0, n, m), rng.integers(0, n, m), n


def g3():
    return np.array([0, 1, 2]), np.array([2, 2, 0]), 3


def operands(rng, n, m, phi, d=2):
    pos = phi.op == "div"
    draw = (lambda r: np.abs(rng.standard_normal((r, d))) + 0.5) if pos else (
        lambda r: rng.standard_normal((r, d)))
    rows = {"src": ("X", n), "dst": ("Y", n), "edge": ("W", m)}
    return {rows[t][0]: draw(rows[t][1]) for t in phi.targets}


def udf_message(phi):
    def msgf(ctx):
        rows = {"src": ctx.src_rows, "dst": ctx.dst_rows, "edge": ctx.edge_rows}
        if phi.op == "copy_lhs":
            return rows[phi.lhs_target]
        if phi.op == "copy_rhs":
            return rows[phi.rhs_target]
        a, b = rows[phi.lhs_target], rows[phi.rhs_target]
        if phi.op == "dot":
            return (a * b).sum(dim=1, keepdim=True)
        return {"add": a + b, "sub": a - b, "mul": a * b, "div": a / b}[phi.op]
    return msgf


def test_udf_all_builtins_match_oracle():
    rng = np.random.default_rng(6000)
    for _ in range(3):
        s, d, n = random_graph(rng, 40, 200, min_nodes=2)
        g = G.from_arrays(s, d, num_nodes=n, device=DEV)
        for phi in kernels.builtin_message_funcs():
            ops = operands(rng, n, s.size, phi)
            for rho in ("sum", "mean", "max", "min"):
                z = G.update_all_udf(g, udf_message(phi), REDUCERS[rho],
                                     src_feat=ops.get("X"), dst_feat=ops.get("Y"),
                                     edge_feat=ops.get("W"))
                want, _ = O.gspmm(s, d, n, phi.op, phi.lhs_target, phi.rhs_target, rho, **ops)
                assert rel_err(to_np(z), want) < 1e-12, (phi.describe(), rho)


def test_udf_matches_fused_kernel():
    rng = np.random.default_rng(6)
    for _ in range(8):
        s, d, n = random_graph(rng, 25, 100, min_nodes=2)
        g = G.from_arrays(s, d, num_nodes=n, device=DEV)
        x = torch.as_tensor(rng.standard_normal((n, 3)), device=DEV)
        w = torch.as_tensor(rng.standard_normal((s.size, 1)), device=DEV)
        z = G.update_all_udf(g, lambda c: c.src_rows * c.edge_rows, lambda b: b.sum(dim=1),
                             src_feat=x, edge_feat=w)
        want, _ = G.gspmm(g, kernels.mul("src", "edge"), "sum", X=x, W=w)
        assert rel_err(to_np(z), to_np(want)) < 1e-12


def test_udf_product_reducer_frozen():
    s, d, n = g3()
    g = G.from_arrays(s, d, num_nodes=n, device=DEV)
    x = np.array([[1.0, 2.0], [3.0, 4.0], [5.0, 6.0]])
    z = G.update_all_udf(g, lambda c: c.src_rows, lambda b: b.prod(dim=1), src_feat=x)
    assert to_np(z).tolist() == [[5.0, 6.0], [0.0, 0.0], [3.0, 8.0]]


def test_udf_dst_rows_available():
    s, d, n = g3()
    g = G.from_arrays(s, d, num_nodes=n, device=DEV)
    x = np.array([[1.0], [2.0], [3.0]])
    z = G.update_all_udf(g, lambda c: c.dst_rows - c.src_rows, lambda b: b.sum(dim=1),
                         src_feat=x, dst_feat=x)
    want, _ = O.gspmm(s, d, n, "sub", "dst", "src", "sum", X=x, Y=x)
    assert np.array_equal(to_np(z), want)


def test_udf_buckets_partition_by_indegree():
    rng = np.random.default_rng(7)
    for _ in range(20):
        s, d, n = random_graph(rng, 40, 160)
        g = G.from_arrays(s, d, num_nodes=n, device=DEV)
        counts = np.bincount(d, minlength=n)
        seen = []

        def reducer(block):
            seen.append(tuple(block.shape))
            return block.sum(dim=1)

        G.update_all_udf(g, lambda c: c.src_rows, reducer, src_feat=np.ones((n, 2)))
        degs = sorted(int(k) for k in np.unique(counts) if k > 0)
        assert [sh[1] for sh in seen] == degs  # ascending, one call per degree
        assert sum(sh[0] for sh in seen) == int((counts > 0).sum())
        for sh, k in zip(seen, degs):
            assert sh == (int((counts == k).sum()), k, 2)


def test_udf_block_rows_ascend_and_follow_csc_order():
    """Bucket rows are destination ids ascending; each row's messages are in
    CSC order (source ascending, then edge id), as the reference's
    adj.edge_ids[indptr[nodes] + arange(k)] gather."""
    s, d, n = np.array([3, 1, 2, 0, 2]), np.array([1, 1, 0, 0, 1]), 4
    g = G.from_arrays(s, d, num_nodes=n, device=DEV)
    eid = torch.arange(5, dtype=torch.float64, device=DEV)[:, None]
    blocks = []

    def reducer(b):
        blocks.append(to_np(b)[..., 0].tolist())
        return b.sum(dim=1)

    G.update_all_udf(g, lambda c: c.edge_rows, reducer, edge_feat=eid)
    # dst 0: edges 3 (src 0), 2 (src 2); dst 1: edges 1 (src 1), 4 (src 2), 0 (src 3)
    assert blocks == [[[3.0, 2.0]], [[1.0, 4.0, 0.0]]]


def test_udf_size_guard_warns():
    n = 1002
    s = np.arange(n - 1)
    g = G.from_arrays(s, s + 1, num_nodes=n, device=DEV)
    x = torch.ones((n, 1000), device=DEV)
    with pytest.warns(RuntimeWarning, match="not fused"):
        G.update_all_udf(g, lambda c: c.src_rows, lambda b: b.sum(dim=1), src_feat=x)


def test_udf_no_warning_under_guard():
    s, d, n = g3()
    g = G.from_arrays(s, d, num_nodes=n, device=DEV)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        G.update_all_udf(g, lambda c: c.src_rows, lambda b: b.sum(dim=1),
                         src_feat=np.ones((3, 1)))


def test_udf_shape_errors():
    s, d, n = g3()
    g = G.from_arrays(s, d, num_nodes=n, device=DEV)
    x = np.ones((3, 2))
    with pytest.raises(ValueError, match="message UDF returned 2 rows"):
        G.update_all_udf(g, lambda c: c.src_rows[:2], lambda b: b.sum(dim=1), src_feat=x)
    with pytest.raises(ValueError, match="reduce UDF returned shape"):
        G.update_all_udf(g, lambda c: c.src_rows, lambda b: b.sum(dim=(1, 2), keepdim=True),
                         src_feat=x)
