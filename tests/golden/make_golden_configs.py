"""Golden outputs of the reference for BASELINE.json configs C1 and C2.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden_configs.py

Inputs are regenerated from seeds by tests/golden/config_inputs.py on both
sides, so only outputs are stored (tests/golden/configs.npz):
  C1  Cora-shaped (n=2708, m=10556) 2-layer mean-GCN [1433, 16, 7], 20
      epochs of full-graph gradient descent (layers.py:137-202): the losses.
  C2  Pubmed-shaped (n=19717, m=88651) 8-head GAT layer 500 -> 8x8
      (layers.py:96-116) with fp32-representable weights: the output (sampled
      rows + column sums) and the gradients of sum(h * U) w.r.t. every
      head's W, a_l, a_r.
"""

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

from config_inputs import SAMPLE_ROWS, c1_inputs, c2_inputs, c2_weights  # noqa: E402


def main():
    import graphmp as G
    from graphmp import autodiff, layers as L

    out = {}
    # ---- C1 ----
    src, dst, n, x, labels = c1_inputs()
    g = G.from_arrays(src.astype(np.uint32), dst.astype(np.uint32), num_nodes=n)
    model = L.GCNModel([1433, 16, 7], seed=0)
    losses = L.train(g, x.astype(np.float64), labels, model, L.TrainConfig(lr=0.05, epochs=20))
    out["c1/losses"] = np.asarray(losses)

    # ---- C2 ----
    src, dst, n, x, u = c2_inputs()
    g = G.from_arrays(src.astype(np.uint32), dst.astype(np.uint32), num_nodes=n)
    params = c2_weights(L.init_gat)
    tape = G.Tape()
    leaves = []
    heads = []
    for hp in params.heads:
        W, al, ar = tape.leaf(hp.W), tape.leaf(hp.a_l), tape.leaf(hp.a_r)
        leaves.append((W, al, ar))
        heads.append(L.GATHead(W=W, a_l=al, a_r=ar))
    h = L.gat_layer(g, x.astype(np.float64), L.GATParams(heads=heads))
    hv = h.value
    prod = _hadamard(h, u.astype(np.float64))
    loss = autodiff.matmul(autodiff.matmul(np.ones((1, n)), prod), np.ones((64, 1)))
    grads = tape.backward(loss)
    out["c2/h_rows"] = hv[SAMPLE_ROWS]
    out["c2/h_colsum"] = hv.sum(axis=0)
    for i, (W, al, ar) in enumerate(leaves):
        out["c2/dW%d" % i] = grads[W]
        out["c2/dal%d" % i] = grads[al]
        out["c2/dar%d" % i] = grads[ar]
    np.savez_compressed(HERE / "configs.npz", **out)
    print("wrote", sorted(out)[:5], "...", len(out))


def _hadamard(a, u):
    tape = a.tape

    def back(up, ctx):
        return [up * ctx["u"]]

    return tape.record("hadamard", (a,), a.value * u, {"u": u}, back)


if __name__ == "__main__":
    main()
