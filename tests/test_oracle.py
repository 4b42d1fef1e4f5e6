"""Pin the CPU oracle against the reference's own outputs (tests/golden/)."""

import numpy as np
import pytest

from conftest import case_operands, golden, golden_graph, golden_meta, rel_err
from oracle import gmp_oracle as O


def _cases():
    return golden_meta()["kernel_cases"]


@pytest.mark.parametrize("chunk", range(8))
def test_oracle_gspmm_gsddmm_match_reference(chunk):
    gd = golden()
    cases = [c for c in _cases() if c["case"] % 8 == chunk]
    for c in cases:
        src, dst, n = golden_graph("g%d" % c["graph"])
        ops = case_operands(c["case"])
        for rho in c["rho"]:
            z, aux = O.gspmm(src, dst, n, c["op"], c["lhs"], c["rhs"], rho, **ops)
            want = gd["c%d/%s/Z" % (c["case"], rho)]
            if rho in ("max", "min"):
                assert np.array_equal(z, want), (c, rho)
                assert np.array_equal(aux, gd["c%d/%s/arg" % (c["case"], rho)]), (c, rho)
            else:
                assert rel_err(z, want) < 1e-12, (c, rho)
            if rho == "mean":
                assert np.array_equal(aux, gd["c%d/mean/counts" % c["case"]])
        m = O.gsddmm(src, dst, n, c["op"], c["lhs"], c["rhs"], **ops)
        assert rel_err(m, gd["c%d/M" % c["case"]]) < 1e-12, c


@pytest.mark.parametrize("chunk", range(4))
def test_oracle_backward_matches_reference(chunk):
    gd = golden()
    key = {"src": "dx", "dst": "dy", "edge": "dw"}
    for c in [c for c in _cases() if c["case"] % 4 == chunk]:
        src, dst, n = golden_graph("g%d" % c["graph"])
        ops = case_operands(c["case"])
        for rho in c["rho"]:
            aux = None
            if rho == "mean":
                aux = gd["c%d/mean/counts" % c["case"]]
            elif rho in ("max", "min"):
                aux = gd["c%d/%s/arg" % (c["case"], rho)]
            grads = O.gspmm_backward(src, dst, n, c["op"], c["lhs"], c["rhs"], rho, aux=aux,
                                     dZ=gd["c%d/%s/dZ" % (c["case"], rho)], **ops)
            for t, g in grads.items():
                want = gd["c%d/%s/%s" % (c["case"], rho, key[t])]
                assert rel_err(g, want) < 1e-10, (c, rho, t)
        grads = O.gsddmm_backward(src, dst, n, c["op"], c["lhs"], c["rhs"],
                                  dM=gd["c%d/dM" % c["case"]], **ops)
        for t, g in grads.items():
            assert rel_err(g, gd["c%d/sddmm/%s" % (c["case"], key[t])]) < 1e-10, (c, t)


def test_oracle_div_by_zero_names_reference_edge():
    gd = golden()
    for rec in golden_meta()["div_zero"]:
        k = rec["k"]
        src, dst, n = golden_graph("dz%d" % k)
        x, w = gd["dz%d/X" % k], gd["dz%d/W" % k]
        for kern, fn in (("gspmm", lambda: O.gspmm(src, dst, n, "div", "src", "edge", "sum",
                                                    X=x, W=w)),
                         ("gsddmm", lambda: O.gsddmm(src, dst, n, "div", "src", "edge",
                                                     X=x, W=w))):
            if rec[kern] is None:
                fn()
            else:
                with pytest.raises(ZeroDivisionError, match="edge id %d$" % rec[kern]):
                    fn()


def test_oracle_edge_softmax_and_backward():
    gd = golden()
    for k in golden_meta()["softmax"]:
        src, dst, n = golden_graph("sm%d" % k)
        s, u = gd["sm%d/s" % k], gd["sm%d/u" % k]
        alpha = O.edge_softmax(src, dst, n, s)
        assert rel_err(alpha, gd["sm%d/alpha" % k]) < 1e-12
        ds = O.edge_softmax_backward(src, dst, n, alpha, u)
        assert rel_err(ds, gd["sm%d/ds" % k]) < 1e-10


def test_oracle_adjacency_bit_exact():
    gd = golden()
    src, dst, n = golden_graph("idx")
    for nm, fn in (("csc", O.csc), ("csr", O.csr)):
        indptr, indices, eids = fn(src, dst, n)
        assert np.array_equal(indptr, gd["idx/%s/indptr" % nm])
        assert np.array_equal(indices, gd["idx/%s/indices" % nm])
        assert np.array_equal(eids, gd["idx/%s/edge_ids" % nm])


def test_reference_frozen_examples():
    """The reference's hand-checked G3 values (test_kernels.py:16-32,
    test_messaging.py:103-109, test_autodiff.py:125-155)."""
    src, dst, n = np.array([0, 1, 2]), np.array([2, 2, 0]), 3
    x = np.array([[1.0], [2.0], [3.0]])
    w = np.array([[10.0], [20.0], [30.0]])
    assert O.gspmm(src, dst, n, "copy_lhs", "src", None, "sum", X=x)[0].tolist() == \
        [[3.0], [0.0], [3.0]]
    assert O.gspmm(src, dst, n, "mul", "src", "edge", "sum", X=x, W=w)[0].tolist() == \
        [[90.0], [0.0], [50.0]]
    z, counts = O.gspmm(src, dst, n, "copy_lhs", "src", None, "mean", X=np.array([[1.], [2.], [4.]]))
    assert counts.tolist() == [1, 0, 2] and z.tolist() == [[4.0], [0.0], [1.5]]
    p = np.array([[1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    assert O.gsddmm(src, dst, n, "dot", "src", "dst", X=p, Y=p).tolist() == [[1.0], [1.0], [1.0]]
    alpha = O.edge_softmax(src, dst, n, np.array([[1.0], [2.0], [3.0]]))
    assert abs(alpha[0, 0] - 0.2689414213699951) < 1e-12
    g = O.gspmm_backward(src, dst, n, "mul", "src", "edge", "sum", X=x, W=w, dZ=np.ones((3, 1)))
    assert g["edge"].tolist() == [[1.0], [2.0], [3.0]]
    assert g["src"].tolist() == [[10.0], [20.0], [30.0]]
    g = O.gspmm_backward(src, dst, n, "copy_lhs", "src", None, "mean", X=np.zeros((3, 1)),
                         aux=np.array([1, 0, 2]), dZ=np.array([[6.0], [7.0], [8.0]]))
    assert g["src"].tolist() == [[4.0], [4.0], [6.0]]


def test_oracle_generators_match_reference():
    from paper_1909_01315_b200 import generators
    gd = golden()
    s, d = generators.power_law_edges(400, 6, seed=3)
    assert np.array_equal(s, gd["gen/power_law_400_6_3/src"])
    assert np.array_equal(d, gd["gen/power_law_400_6_3/dst"])
    s, d = generators.constant_indegree_edges(200, 5, seed=2)
    assert np.array_equal(s, gd["gen/constant_indegree_200_5_2/src"])
    assert np.array_equal(d, gd["gen/constant_indegree_200_5_2/dst"])
