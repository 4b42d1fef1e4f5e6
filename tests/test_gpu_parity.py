"""Parity of the CUDA kernels with the reference (golden fixtures) and the
oracle (larger graphs). Every call here goes through libgmp.so.

Bars (north star): integer / index outputs and max/min values bit-exact;
sum / mean / softmax within rtol 1e-5, atol 1e-6 in fp32. The fp64
instantiation is held to the reference's own 1e-12 relative bound.
"""

import threading

import numpy as np
import pytest
import torch

import paper_1909_01315_b200 as G
from paper_1909_01315_b200 import _lib, kernels
from conftest import (assert_close32, case_operands, golden, golden_graph, golden_meta,
                      rel_err, to_np)
from oracle import gmp_oracle as O

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _phi(c):
    return kernels.MessageFunc(c["op"], c["lhs"], c["rhs"])


def _dev(ops, dtype):
    return {k: torch.as_tensor(v, device=DEV).to(dtype) for k, v in ops.items()}


@pytest.fixture(scope="module")
def golden_graphs():
    out = {}
    for gi in range(8):
        src, dst, n = golden_graph("g%d" % gi)
        out[gi] = G.from_arrays(src.astype(np.int64), dst.astype(np.int64), num_nodes=n,
                                device=DEV)
    return out


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_gspmm_all_phi_rho_vs_reference(golden_graphs, dtype):
    gd = golden()
    n_checked = 0
    for c in golden_meta()["kernel_cases"]:
        g = golden_graphs[c["graph"]]
        phi = _phi(c)
        ops = _dev(case_operands(c["case"]), dtype)
        for rho in c["rho"]:
            z, aux = G.gspmm(g, phi, rho, **ops)
            assert z.dtype == dtype
            z = to_np(z)
            want = gd["c%d/%s/Z" % (c["case"], rho)]
            tag = (c, rho, str(dtype))
            if rho in ("max", "min"):
                if dtype == torch.float64:
                    assert np.array_equal(z, want), tag
                else:
                    assert np.array_equal(z, want.astype(np.float32)), tag
                assert np.array_equal(to_np(aux.arg_edge), gd["c%d/%s/arg" % (c["case"], rho)]), tag
            elif dtype == torch.float64:
                assert rel_err(z, want) < 1e-12, tag
            else:
                assert_close32(z, want, str(tag))
            if rho == "mean":
                assert np.array_equal(to_np(aux), gd["c%d/mean/counts" % c["case"]]), tag
            n_checked += 1
    assert n_checked == 4 * len(golden_meta()["kernel_cases"])


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_gsddmm_all_phi_vs_reference(golden_graphs, dtype):
    gd = golden()
    for c in golden_meta()["kernel_cases"]:
        g = golden_graphs[c["graph"]]
        phi = _phi(c)
        m = to_np(G.gsddmm(g, phi, **_dev(case_operands(c["case"]), dtype)))
        want = gd["c%d/M" % c["case"]]
        if phi.op == "dot":
            if dtype == torch.float64:
                assert rel_err(m, want) < 1e-12, c
            else:
                assert_close32(m, want, str(c))
        elif dtype == torch.float64:
            assert np.array_equal(m, want), c
        else:  # fp64 message rounded once == the reference's result rounded
            assert np.array_equal(m, want.astype(np.float32)), c


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_backward_vs_reference(golden_graphs, dtype):
    gd = golden()
    key = {"x": "dx", "y": "dy", "w": "dw"}
    for c in golden_meta()["kernel_cases"]:
        g = golden_graphs[c["graph"]]
        phi = _phi(c)
        ops = _dev(case_operands(c["case"]), dtype)
        needs = tuple(k.lower() for k in ops)
        for rho in c["rho"]:
            z, aux = G.gspmm(g, phi, rho, **ops)
            dz = torch.as_tensor(gd["c%d/%s/dZ" % (c["case"], rho)], device=DEV).to(dtype)
            b = G.gspmm_backward(g, phi, rho, **ops, aux=aux, dZ=dz, needs=needs)
            for nd in needs:
                want = gd["c%d/%s/%s" % (c["case"], rho, key[nd])]
                got = to_np(getattr(b, key[nd]))
                if dtype == torch.float64:
                    assert rel_err(got, want) < 1e-10, (c, rho, nd)
                else:
                    assert_close32(got, want, str((c, rho, nd)))
        dm = torch.as_tensor(gd["c%d/dM" % c["case"]], device=DEV).to(dtype)
        b = G.gsddmm_backward(g, phi, **ops, dM=dm, needs=needs)
        for nd in needs:
            want = gd["c%d/sddmm/%s" % (c["case"], key[nd])]
            got = to_np(getattr(b, key[nd]))
            if dtype == torch.float64:
                assert rel_err(got, want) < 1e-10, (c, nd)
            else:
                assert_close32(got, want, str((c, nd)))


def test_div_by_zero_names_reference_edge():
    gd = golden()
    for rec in golden_meta()["div_zero"]:
        k = rec["k"]
        src, dst, n = golden_graph("dz%d" % k)
        g = G.from_arrays(src.astype(np.int64), dst.astype(np.int64), n, device=DEV)
        x = torch.as_tensor(gd["dz%d/X" % k], device=DEV)
        w = torch.as_tensor(gd["dz%d/W" % k], device=DEV)
        for kern in ("gspmm", "gsddmm"):
            def call():
                if kern == "gspmm":
                    return G.gspmm(g, kernels.div("src", "edge"), "sum", X=x, W=w)
                return G.gsddmm(g, kernels.div("src", "edge"), X=x, W=w)
            if rec[kern] is None:
                call()
            else:
                with pytest.raises(ZeroDivisionError, match="edge id %d$" % rec[kern]):
                    call()


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_edge_softmax_vs_reference(dtype):
    gd = golden()
    for k in golden_meta()["softmax"]:
        src, dst, n = golden_graph("sm%d" % k)
        g = G.from_arrays(src.astype(np.int64), dst.astype(np.int64), n, device=DEV)
        s = torch.as_tensor(gd["sm%d/s" % k], device=DEV).to(dtype).requires_grad_(True)
        u = torch.as_tensor(gd["sm%d/u" % k], device=DEV).to(dtype)
        alpha = G.edge_softmax(g, s)
        (alpha * u).sum().backward()
        if dtype == torch.float64:
            assert rel_err(to_np(alpha), gd["sm%d/alpha" % k]) < 1e-12
            assert rel_err(to_np(s.grad), gd["sm%d/ds" % k]) < 1e-10
        else:
            assert_close32(alpha, gd["sm%d/alpha" % k], "alpha sm%d" % k)
            assert_close32(s.grad, gd["sm%d/ds" % k], "ds sm%d" % k)


def test_frozen_reference_examples():
    g = G.build_graph(3, [(0, 2), (1, 2), (2, 0)], device=DEV)
    x = np.array([[1.0], [2.0], [3.0]])
    w = np.array([[10.0], [20.0], [30.0]])
    z, aux = G.gspmm(g, kernels.copy("src"), "sum", X=x)
    assert z.tolist() == [[3.0], [0.0], [3.0]] and aux is None
    z, _ = G.gspmm(g, kernels.mul("src", "edge"), "sum", X=x, W=w)
    assert z.tolist() == [[90.0], [0.0], [50.0]]
    p = np.array([[1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    assert G.gsddmm(g, kernels.dot("src", "dst"), X=p, Y=p).tolist() == [[1.0], [1.0], [1.0]]
    z, aux = G.gspmm(g, kernels.copy("src"), "mean", X=np.array([[1.], [2.], [4.]]))
    assert to_np(aux).tolist() == [1, 0, 2] and z.tolist() == [[4.0], [0.0], [1.5]]
    z, aux = G.gspmm(g, kernels.copy("src"), "max", X=np.array([[1.], [2.], [4.]]))
    assert z[1].tolist() == [0.0] and aux.arg_edge[1].tolist() == [-1]
    assert aux.arg_edge[0].tolist() == [2] and bool(aux.empty_rows[1])
    gt = G.build_graph(2, [(0, 1), (0, 1), (0, 1)], device=DEV)
    for strat in kernels.GSPMM_STRATEGIES:
        z, aux = G.gspmm(gt, kernels.copy_rhs("edge"), "max", W=np.full((3, 1), 5.0),
                         strategy=strat, fmt="coo" if strat == "serial_reference" else None)
        assert float(z[1, 0]) == 5.0 and int(aux.arg_edge[1, 0]) == 0
    alpha = G.edge_softmax(g, np.array([[1.0], [2.0], [3.0]]))
    assert abs(float(alpha[0, 0]) - 0.2689414213699951) < 1e-12
    g2 = G.build_graph(2, [(0, 0), (0, 1)], device=DEV)
    m = G.gsddmm(g2, kernels.sub("dst", "src"), X=np.array([[3.0, 1.0], [7.0, 2.0]]),
                 Y=np.array([[3.0, 1.0], [7.0, 2.0]]))
    assert m.tolist() == [[0.0, 0.0], [4.0, 1.0]]


def test_empty_and_degenerate_shapes():
    g = G.build_graph(4, [], device=DEV)
    z, _ = G.gspmm(g, kernels.copy("src"), "sum", X=torch.ones(4, 3, device=DEV))
    assert tuple(z.shape) == (4, 3) and not bool(z.any())
    z, aux = G.gspmm(g, kernels.copy("src"), "max", X=torch.ones(4, 3, device=DEV))
    assert not bool(z.any()) and bool((aux.arg_edge == -1).all())
    m = G.gsddmm(g, kernels.copy("src"), X=torch.ones(4, 3, device=DEV))
    assert tuple(m.shape) == (0, 3)
    m = G.gsddmm(g, kernels.mul("src", "edge"), X=torch.ones(4, 3, device=DEV),
                 W=torch.ones(0, 1, device=DEV))
    assert tuple(m.shape) == (0, 3)
    g0 = G.build_graph(0, [], device=DEV)
    z, _ = G.gspmm(g0, kernels.copy("src"), "sum", X=torch.ones(0, 2, device=DEV))
    assert tuple(z.shape) == (0, 2)
    g3 = G.build_graph(3, [(0, 2), (1, 2)], device=DEV)
    z, cnt = G.gspmm(g3, kernels.copy("src"), "mean", X=torch.ones(3, 0, device=DEV))
    assert tuple(z.shape) == (3, 0) and to_np(cnt).tolist() == [0, 0, 2]


def _power_law_graph(n, deg, seed):
    s, d = G.generators.power_law_edges(n, deg, seed)
    return s, d, G.from_arrays(s, d, num_nodes=n, device=DEV)


@pytest.mark.parametrize("d", [1, 2, 3, 16, 64, 100, 256, 602])
def test_power_law_heavy_rows_vs_oracle(d):
    """Power-law in-degrees: hub rows take the CTA path, the rest the warp
    path; fp32 inputs, every reducer, copy_u and u_mul_e (scalar w)."""
    n, deg = (6000, 40) if d >= 256 else (20000, 40)
    s, dd, g = _power_law_graph(n, deg, 7)
    sched = g.to_csc().schedule()
    assert sched.n_heavy > 0
    rng = np.random.default_rng(d)
    x = rng.standard_normal((n, d)).astype(np.float32)
    w = rng.standard_normal((s.size, 1)).astype(np.float32)
    adj = O.csc(s, dd, n)
    xt, wt = torch.as_tensor(x, device=DEV), torch.as_tensor(w, device=DEV)
    for phi, kw, kwo in ((kernels.copy("src"), {"X": xt}, ("copy_lhs", "src", None, {"X": x})),
                         (kernels.mul("src", "edge"), {"X": xt, "W": wt},
                          ("mul", "src", "edge", {"X": x, "W": w}))):
        for rho in ("sum", "mean", "max", "min"):
            z, aux = G.gspmm(g, phi, rho, **kw)
            want, waux = O.gspmm(s, dd, n, kwo[0], kwo[1], kwo[2], rho, adj=adj, workers=8, **kwo[3])
            if rho in ("max", "min"):
                assert np.array_equal(to_np(z), want.astype(np.float32)), (d, rho)
                assert np.array_equal(to_np(aux.arg_edge), waux), (d, rho)
            else:
                assert_close32(z, want, "d=%d %s %s" % (d, phi.describe(), rho))


def test_single_hub_row_and_tiles():
    """All edges into node 0 (one CTA row) plus forced narrow column tiles."""
    m, n, d = 100_000, 500, 48
    rng = np.random.default_rng(3)
    s = rng.integers(0, n, m)
    dd = np.zeros(m, dtype=np.int64)
    dd[::97] = rng.integers(1, n, dd[::97].size)
    g = G.from_arrays(s, dd, n, device=DEV)
    x = rng.standard_normal((n, d)).astype(np.float32)
    want, _ = O.gspmm(s, dd, n, "copy_lhs", "src", None, "sum", X=x)
    wmax, warg = O.gspmm(s, dd, n, "copy_lhs", "src", None, "max", X=x)
    for tc in (None, 8, 16, 24):
        with kernels.tuning(tile_cols=tc):
            z, _ = G.gspmm(g, kernels.copy("src"), "sum", X=torch.as_tensor(x, device=DEV))
            zm, am = G.gspmm(g, kernels.copy("src"), "max", X=torch.as_tensor(x, device=DEV))
        assert_close32(z, want, "tile %s" % tc)
        assert np.array_equal(to_np(zm), wmax.astype(np.float32))
        assert np.array_equal(to_np(am.arg_edge), warg)


def test_strided_and_unaligned_operands():
    rng = np.random.default_rng(11)
    n, m = 300, 5000
    s, dd = rng.integers(0, n, m), rng.integers(0, n, m)
    g = G.from_arrays(s, dd, n, device=DEV)
    big = torch.as_tensor(rng.standard_normal((n, 13)).astype(np.float32), device=DEV)
    wbig = torch.as_tensor(rng.standard_normal((m, 7)).astype(np.float32), device=DEV)
    for c0, c1 in ((1, 4), (0, 6), (3, 11), (2, 3)):
        x = big[:, c0:c1]
        xw = wbig[:, 0:c1 - c0] if c1 - c0 <= 7 else None
        want, _ = O.gspmm(s, dd, n, "copy_lhs", "src", None, "sum", X=to_np(x))
        z, _ = G.gspmm(g, kernels.copy("src"), "sum", X=x)
        assert_close32(z, want, "view %d:%d" % (c0, c1))
        if xw is not None:
            wantm = O.gsddmm(s, dd, n, "add", "src", "edge", X=to_np(x), W=to_np(xw))
            mm = G.gsddmm(g, kernels.add("src", "edge"), X=x, W=xw)
            assert np.array_equal(to_np(mm), wantm.astype(np.float32))


def test_deterministic_bitwise():
    s, dd, g = _power_law_graph(20000, 40, 1)
    x = torch.randn(20000, 32, device=DEV)
    a, _ = G.gspmm(g, kernels.copy("src"), "sum", X=x)
    b, _ = G.gspmm(g, kernels.copy("src"), "sum", X=x)
    assert torch.equal(a, b)


def test_concurrent_calls_share_graph():
    rng = np.random.default_rng(8)
    n, m = 400, 4000
    g = G.from_arrays(rng.integers(0, n, m), rng.integers(0, n, m), n, device=DEV)
    x = torch.as_tensor(rng.standard_normal((n, 4)), device=DEV)
    want, _ = G.gspmm(g, kernels.copy("src"), "sum", X=x)
    outs = [None] * 6

    def run(i):
        with torch.cuda.stream(torch.cuda.Stream()):
            outs[i] = G.gspmm(g, kernels.copy("src"), "sum", X=x)[0]
            torch.cuda.current_stream().synchronize()

    ts = [threading.Thread(target=run, args=(i,)) for i in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for o in outs:
        assert torch.equal(o, want)


def test_fusion_memory_bound_and_dispatch_log():
    rng = np.random.default_rng(2)
    n, m, d = 50, 60000, 8
    g = G.from_arrays(rng.integers(0, n, m), rng.integers(0, n, m), n, device=DEV)
    g.to_csc().schedule()
    x = torch.as_tensor(rng.standard_normal((n, d)), device=DEV)
    w = torch.as_tensor(rng.standard_normal((m, d)), device=DEV)
    edge_bytes = m * d * 8
    for rho in ("sum", "max", "mean"):
        with G.track_allocations() as meter:
            G.gspmm(g, kernels.mul("src", "edge"), rho, X=x, W=w)
        assert meter.peak_bytes < edge_bytes and meter.largest_single_bytes < edge_bytes
        assert meter.peak_bytes <= 3 * n * d * 8
    with G.capture_dispatch() as log:
        G.gspmm(g, kernels.copy("src"), "sum", X=x)
        G.gsddmm(g, kernels.dot("src", "dst"), X=x, Y=x)
    assert [r.kernel for r in log] == ["gspmm", "gsddmm"]
    assert log[0].phi == "copy_lhs(src)" and log[0].graph_id == g.uid and log[1].rows == m


def test_native_library_is_what_runs():
    """The kernels launch through libgmp.so (launch counter moves)."""
    before = _lib.launch_count()
    g = G.build_graph(3, [(0, 2), (1, 2), (2, 0)], device=DEV)
    G.gspmm(g, kernels.copy("src"), "sum", X=torch.ones(3, 2, device=DEV))
    G.gsddmm(g, kernels.copy("src"), X=torch.ones(3, 2, device=DEV))
    assert _lib.launch_count() >= before + 2


@pytest.mark.parametrize("d", [4, 16, 32, 64])
def test_edge_operand_extrema_medium_rows(d):
    """max / min of copy_lhs(edge) (and of an edge-keyed binary message) on a
    power-law graph whose medium and heavy rows take the 256 B-row kernels:
    the operand is gathered by edge id, never by the neighbour id the
    pipelined copy_u ring uses (C5 sweep regression: rows of degree >= 33
    returned the extrema of the wrong rows at d = 16 / 32 / 64)."""
    s, dd, g = _power_law_graph(60000, 20, 0)
    n = 60000
    rng = np.random.default_rng(d)
    w = (np.abs(rng.standard_normal((s.size, d))) + 0.5).astype(np.float32)
    x = (np.abs(rng.standard_normal((n, d))) + 0.5).astype(np.float32)
    adj = O.csc(s, dd, n)
    wt, xt = torch.as_tensor(w, device=DEV), torch.as_tensor(x, device=DEV)
    for phi, kw, kwo in ((kernels.copy("edge"), {"W": wt}, ("copy_lhs", "edge", None, {"W": w})),
                         (kernels.mul("src", "edge"), {"X": xt, "W": wt},
                          ("mul", "src", "edge", {"X": x, "W": w}))):
        for rho in ("max", "min"):
            z, aux = G.gspmm(g, phi, rho, **kw)
            want, waux = O.gspmm(s, dd, n, kwo[0], kwo[1], kwo[2], rho, adj=adj, workers=8, **kwo[3])
            assert np.array_equal(to_np(z), want.astype(np.float32)), (d, phi.describe(), rho)
            assert np.array_equal(to_np(aux.arg_edge), waux), (d, phi.describe(), rho)
