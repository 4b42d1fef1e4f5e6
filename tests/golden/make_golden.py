"""Generate the golden parity fixtures by running the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports graphmp from /root/reference/pkg/src and records inputs + outputs
of gspmm / gsddmm / edge_softmax / gspmm_backward / gsddmm_backward, the
CSC/CSR index arrays and power_law edge lists into tests/golden/*.npz. All
feature inputs are drawn as float32 and stored as float32, so the same bytes
feed the fp32 kernels; the reference computes on their exact float64 upcast.
Nothing at test or bench time reads /root/reference.
"""

import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent


def _ref():
    sys.path.insert(0, REF)
    import graphmp as G
    from graphmp import autodiff, kernels
    return G, autodiff, kernels


def _draw(rng, rows, d, positive):
    a = rng.standard_normal((rows, d)).astype(np.float32)
    if positive:
        a = (np.abs(a) + 0.5).astype(np.float32)
    return a


def _operands(rng, g, phi, d, positive, bcast=None):
    """Operands for phi; bcast in {None, 'lhs', 'rhs'} gives that side 1 column."""
    ops = {}
    for slot, target in (("X", "src"), ("Y", "dst"), ("W", "edge")):
        if target in phi.targets:
            rows = g.num_edges if target == "edge" else g.num_nodes
            width = d
            if bcast == "lhs" and target == phi.lhs_target:
                width = 1
            if bcast == "rhs" and target == phi.rhs_target:
                width = 1
            ops[slot] = _draw(rng, rows, width, positive)
    return ops


def _rand_graph(G, rng, max_nodes, max_edges, min_nodes=1):
    n = int(rng.integers(min_nodes, max_nodes + 1))
    m = int(rng.integers(0, max_edges + 1))
    src = rng.integers(0, n, size=m).astype(np.uint32)
    dst = rng.integers(0, n, size=m).astype(np.uint32)
    return G.from_arrays(src, dst, num_nodes=n)


def main():
    G, autodiff, kernels = _ref()
    rng = np.random.default_rng(20260917)
    store = {}
    meta = []

    def put(key, arr):
        store[key] = np.asarray(arr)

    # --- kernel cases: random multigraphs x 30 phi x 4 rho (+ broadcast) ------
    case = 0
    graphs = [_rand_graph(G, rng, 24, 96) for _ in range(6)]
    graphs.append(G.build_graph(4, []))                       # empty graph
    graphs.append(G.from_arrays(np.arange(300, dtype=np.uint32) % 7,
                                np.zeros(300, dtype=np.uint32), num_nodes=9))  # hub + empties
    for gi, g in enumerate(graphs):
        src, dst, _ = g.coo()
        put("g%d/src" % gi, src)
        put("g%d/dst" % gi, dst)
        put("g%d/n" % gi, np.int64(g.num_nodes))
        for phi in kernels.builtin_message_funcs():
            variants = [None] if phi.op in ("copy_lhs", "copy_rhs", "dot") else [None, "lhs", "rhs"]
            for bc in variants:
                d = 3 if bc is None else 4
                ops = _operands(rng, g, phi, d, positive=phi.op == "div", bcast=bc)
                ops64 = {k: v.astype(np.float64) for k, v in ops.items()}
                rec = {"case": case, "graph": gi, "op": phi.op, "lhs": phi.lhs_target,
                       "rhs": phi.rhs_target, "bcast": bc, "rho": []}
                for k, v in ops.items():
                    put("c%d/%s" % (case, k), v)
                for rho in ("sum", "mean", "max", "min"):
                    z, aux = G.gspmm(g, phi, rho, **ops64)
                    put("c%d/%s/Z" % (case, rho), z)
                    if rho == "mean":
                        put("c%d/mean/counts" % case, aux)
                    if rho in ("max", "min"):
                        put("c%d/%s/arg" % (case, rho), aux.arg_edge)
                    dz = rng.standard_normal(z.shape).astype(np.float32)
                    needs = tuple(k.lower() for k in ops)
                    b = G.gspmm_backward(g, phi, rho, **ops64, aux=aux,
                                         dZ=dz.astype(np.float64), needs=needs)
                    put("c%d/%s/dZ" % (case, rho), dz)
                    for nm in ("dx", "dy", "dw"):
                        v = getattr(b, nm)
                        if v is not None:
                            put("c%d/%s/%s" % (case, rho, nm), v)
                    rec["rho"].append(rho)
                m_out = G.gsddmm(g, phi, **ops64)
                put("c%d/M" % case, m_out)
                dm = rng.standard_normal(m_out.shape).astype(np.float32)
                needs = tuple(k.lower() for k in ops)
                b = G.gsddmm_backward(g, phi, **ops64, dM=dm.astype(np.float64), needs=needs)
                put("c%d/dM" % case, dm)
                for nm in ("dx", "dy", "dw"):
                    v = getattr(b, nm)
                    if v is not None:
                        put("c%d/sddmm/%s" % (case, nm), v)
                meta.append(rec)
                case += 1

    # --- div-by-zero: which edge id the reference names ----------------------
    divz = []
    for k in range(4):
        g = _rand_graph(G, rng, 16, 60, min_nodes=4)
        if g.num_edges == 0:
            continue
        x = _draw(rng, g.num_nodes, 2, True)
        w = _draw(rng, g.num_edges, 2, True)
        zero_e = rng.choice(g.num_edges, size=min(3, g.num_edges), replace=False)
        w[zero_e, int(rng.integers(0, 2))] = 0.0
        src, dst, _ = g.coo()
        rec = {"k": k}
        for kern in ("gspmm", "gsddmm"):
            try:
                if kern == "gspmm":
                    G.gspmm(g, kernels.div("src", "edge"), "sum", X=x.astype(np.float64),
                            W=w.astype(np.float64))
                else:
                    G.gsddmm(g, kernels.div("src", "edge"), X=x.astype(np.float64),
                             W=w.astype(np.float64))
                rec[kern] = None
            except ZeroDivisionError as exc:
                rec[kern] = int(str(exc).rsplit(" ", 1)[1])
        put("dz%d/src" % k, src)
        put("dz%d/dst" % k, dst)
        put("dz%d/n" % k, np.int64(g.num_nodes))
        put("dz%d/X" % k, x)
        put("dz%d/W" % k, w)
        divz.append(rec)

    # --- edge softmax: forward and gradient of sum(alpha * U) -----------------
    sm = []
    for k in range(6):
        g = _rand_graph(G, rng, 30, 150, min_nodes=2)
        H = [1, 1, 3, 8, 2, 5][k]
        s = (rng.standard_normal((g.num_edges, H)) * [1, 50, 3, 2, 10, 1][k]).astype(np.float32)
        u = rng.standard_normal((g.num_edges, H)).astype(np.float32)
        alpha = G.edge_softmax(g, s.astype(np.float64))
        tape = G.Tape()
        sv = tape.leaf(s.astype(np.float64))
        a = G.edge_softmax(g, sv)
        flat = autodiff.matmul(autodiff.matmul(np.ones((1, g.num_edges)),
                                               _hadamard(autodiff, a, u.astype(np.float64))),
                               np.ones((H, 1)))
        grads = tape.backward(flat)
        src, dst, _ = g.coo()
        put("sm%d/src" % k, src)
        put("sm%d/dst" % k, dst)
        put("sm%d/n" % k, np.int64(g.num_nodes))
        put("sm%d/s" % k, s)
        put("sm%d/u" % k, u)
        put("sm%d/alpha" % k, alpha)
        put("sm%d/ds" % k, grads[sv])
        sm.append(k)

    # --- graph indexes and generators ----------------------------------------
    g = _rand_graph(G, rng, 40, 400, min_nodes=10)
    src, dst, _ = g.coo()
    c, r = g.to_csc(), g.to_csr()
    put("idx/src", src)
    put("idx/dst", dst)
    put("idx/n", np.int64(g.num_nodes))
    for nm, adj in (("csc", c), ("csr", r)):
        put("idx/%s/indptr" % nm, adj.indptr)
        put("idx/%s/indices" % nm, adj.indices)
        put("idx/%s/edge_ids" % nm, adj.edge_ids)
    pl = G.power_law(400, 6, seed=3)
    put("gen/power_law_400_6_3/src", pl.src)
    put("gen/power_law_400_6_3/dst", pl.dst)
    ci = G.constant_indegree(200, 5, seed=2)
    put("gen/constant_indegree_200_5_2/src", ci.src)
    put("gen/constant_indegree_200_5_2/dst", ci.dst)

    # --- layers: 2-layer mean-GCN losses and a GAT layer on small graphs ------
    from graphmp import layers as L
    g = _rand_graph(G, rng, 60, 400, min_nodes=30)
    x = rng.standard_normal((g.num_nodes, 12)).astype(np.float32)
    labels = rng.integers(0, 3, size=g.num_nodes)
    model = L.GCNModel([12, 8, 3], seed=0)
    losses = L.train(g, x.astype(np.float64), labels, model, L.TrainConfig(lr=0.1, epochs=5))
    src, dst, _ = g.coo()
    put("gcn/src", src)
    put("gcn/dst", dst)
    put("gcn/n", np.int64(g.num_nodes))
    put("gcn/x", x)
    put("gcn/labels", labels)
    put("gcn/losses", np.asarray(losses))
    params = L.init_gat(np.random.default_rng(1), 12, 4, 3)
    h = L.gat_layer(g, x.astype(np.float64), params)
    put("gat/out", h)

    np.savez_compressed(OUT / "reference_cases.npz", **store)
    (OUT / "reference_cases.json").write_text(json.dumps(
        {"kernel_cases": meta, "div_zero": divz, "softmax": sm,
         "generator": "tests/golden/make_golden.py", "reference": "graphmp 0.1.0 @ " + REF},
        indent=0))
    print("wrote %d arrays, %d kernel cases" % (len(store), len(meta)))


def _hadamard(autodiff, a, u):
    """a * u for a taped a and a constant u, via the reference's tape."""
    av = a.value
    out = av * u
    tape = a.tape

    def back(up, ctx):
        return [up * ctx["u"]]

    return tape.record("hadamard", (a,), out, {"u": u}, back)


if __name__ == "__main__":
    main()
