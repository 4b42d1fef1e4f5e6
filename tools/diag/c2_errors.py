"""Elementwise error report of the C2 (Pubmed-shaped 8-head GAT layer) fp32
forward/backward against the reference goldens: how far each output is from
north_star's rtol 1e-5 / atol 1e-6 bar, and which part of the layer (the
sparse path vs the dense cuBLAS projections) the error comes from."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))
import paper_1909_01315_b200 as G  # noqa: E402
from paper_1909_01315_b200 import layers  # noqa: E402
from config_inputs import SAMPLE_ROWS, c2_inputs, c2_weights  # noqa: E402


def report(name, got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    d = np.abs(got - want)
    bad = ~np.isclose(got, want, rtol=1e-5, atol=1e-6)
    # the atol that would make every cell pass at rtol 1e-5
    need = np.max(np.maximum(d - 1e-5 * np.abs(want), 0))
    print("%-10s cells=%7d outside=%5d max|d|=%.3g max|want|=%.3g atol_needed=%.3g" % (
        name, d.size, bad.sum(), d.max(), np.abs(want).max(), need))


def main():
    torch.backends.cuda.matmul.allow_tf32 = False
    gold = dict(np.load(ROOT / "tests" / "golden" / "configs.npz"))
    src, dst, n, x, u = c2_inputs()
    g = G.from_arrays(src, dst, num_nodes=n, device="cuda")
    for fused, dense in ((True, "fp32"), (False, "fp32"), (True, "fp64"), (False, "fp64")):
        params = c2_weights(layers.init_gat)
        leaves = []
        for hp in params.heads:
            hp.W, hp.a_l, hp.a_r = (torch.as_tensor(a, device="cuda").float().requires_grad_(True)
                                    for a in (hp.W, hp.a_l, hp.a_r))
            leaves.append((hp.W, hp.a_l, hp.a_r))
        xt = torch.as_tensor(x, device="cuda").float()
        with layers.dense_precision(dense):
            h = layers.gat_layer(g, xt, params, fused=fused)
            (h * torch.as_tensor(u, device="cuda").float()).sum().backward()
        print("fused=%s dense=%s" % (fused, dense))
        report("h_rows", h.detach().cpu().numpy()[SAMPLE_ROWS], gold["c2/h_rows"])
        for i, (W, al, ar) in enumerate(leaves[:3]):
            report("dW%d" % i, W.grad.cpu().numpy(), gold["c2/dW%d" % i])
            report("dal%d" % i, al.grad.cpu().numpy(), gold["c2/dal%d" % i])
            report("dar%d" % i, ar.grad.cpu().numpy(), gold["c2/dar%d" % i])


if __name__ == "__main__":
    main()
