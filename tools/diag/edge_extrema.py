"""Repro: copy_lhs(edge) max/min on the C5 power-law graph vs the oracle
(per-row degree of the mismatching rows)."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1909_01315_b200 as G  # noqa: E402
from paper_1909_01315_b200 import kernels  # noqa: E402
from oracle import gmp_oracle as O  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
s, d = G.generators.power_law_edges(n, 20, seed=0)
g = G.from_arrays(s, d, num_nodes=n, device="cuda")
adj = g.to_csc()
sched = adj.schedule()
print("n", n, "m", s.size, "heavy", sched.n_heavy, "max_deg", int(adj.degrees().max()))
deg = np.bincount(d, minlength=n)
for dim in (4, 16, 32):
    gen = torch.Generator(device="cuda"); gen.manual_seed(dim)
    W = torch.randn((s.size, dim), generator=gen, device="cuda").abs() + 0.5
    for rho in ("max",):
        z, aux = G.gspmm(g, kernels.copy("edge"), rho, W=W)
        want, warg = O.gspmm(s, d, n, "copy_lhs", "edge", None, rho, W=W.cpu().numpy(), workers=8)
        got = z.cpu().numpy()
        bad = np.flatnonzero((got != want.astype(np.float32)).any(axis=1))
        print(dim, rho, "bad rows", bad.size, "degrees", np.unique(deg[bad])[:10], "max|d|",
              float(np.abs(got - want).max()))
        if bad.size:
            r = bad[0]
            print("  row", r, "deg", deg[r], "got", got[r][:4], "want", want[r][:4])
