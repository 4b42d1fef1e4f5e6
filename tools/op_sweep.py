"""Op sweep (BASELINE.json config C5): every built-in phi x rho for g-SpMM and
every phi for g-SDDMM, feature dims 1..512, uniform vs power-law graphs.

Writes a CSV in the reference bench schema (bench.py:39-41 COLUMNS:
kernel,phi,rho,strategy,format,num_nodes,num_edges,feat_size,heads,repeats,
median_seconds,gflops,peak_aux_bytes) extended with graph, gbps (algorithmic
bytes, SURVEY 8(d) model) and roofline_frac (of MEASURED_PEAKS hbm_gbs).
gflops uses the reference's continuity formula 2 * m * d (bench.py:146).

    python tools/op_sweep.py --nodes 1000000 --out profiles/r01_op_sweep.csv
"""

import argparse
import csv
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_1909_01315_b200 as G  # noqa: E402
from paper_1909_01315_b200 import kernels  # noqa: E402

COLUMNS = ("kernel", "phi", "rho", "strategy", "format", "num_nodes", "num_edges", "feat_size",
           "heads", "repeats", "median_seconds", "gflops", "peak_aux_bytes", "graph", "gbps",
           "roofline_frac")


def op_bytes(kind, phi, rho, n, m, shapes, d_out, F):
    """Algorithmic bytes: indices + every operand read once per use + outputs."""
    b = 0
    if kind == "gspmm":
        b += (n + 1) * 8 + m * 4
        uses_eid = "edge" in phi.targets or rho in ("max", "min")
        b += m * 4 if uses_eid else 0
        for t in phi.targets:
            w = shapes[t]
            b += (n if t == "dst" else m) * w * F
        b += n * d_out * F + (n * d_out * 8 if rho in ("max", "min") else 0)
    else:
        b += 2 * m * 4
        for t in phi.targets:
            b += m * shapes[t] * F
        b += m * d_out * F
    return b


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--nodes", type=int, default=1_000_000)
    p.add_argument("--deg", type=int, default=20)
    p.add_argument("--dims", default="1,2,4,8,16,32,64,128,256,512")
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--out", default="gpurun_out/op_sweep.csv")
    p.add_argument("--quick", action="store_true", help="one phi per op family")
    a = p.parse_args()
    dev = torch.device("cuda")
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    n = a.nodes
    rng = np.random.default_rng(0)
    graphs = {
        "power_law": G.generators.power_law_edges(n, a.deg, seed=0),
        "uniform": (rng.integers(0, n, n * a.deg), rng.integers(0, n, n * a.deg)),
    }
    phis = kernels.builtin_message_funcs()
    if a.quick:
        keep = {"copy_lhs(src)", "copy_lhs(edge)", "mul(src,edge)", "add(src,dst)",
                "sub(edge,dst)", "div(src,edge)", "dot(src,dst)"}
        phis = [f for f in phis if f.describe() in keep]
    rows = []
    for gname, (s, d) in graphs.items():
        g = G.from_arrays(s, d, num_nodes=n, device=dev)
        g.to_csc().schedule()
        m = g.num_edges
        for dim in [int(x) for x in a.dims.split(",")]:
            gen = torch.Generator(device=dev)
            gen.manual_seed(dim)
            X = torch.randn((n, dim), generator=gen, device=dev).abs() + 0.5  # div-safe
            Y = torch.randn((n, dim), generator=gen, device=dev).abs() + 0.5
            W = torch.randn((m, dim), generator=gen, device=dev).abs() + 0.5
            ops = {"src": ("X", X), "dst": ("Y", Y), "edge": ("W", W)}
            for phi in phis:
                kw = {ops[t][0]: ops[t][1] for t in phi.targets}
                shapes = {t: dim for t in phi.targets}
                d_out = 1 if phi.op == "dot" else dim
                for rho in ("sum", "mean", "max", "min"):
                    t = timeit(lambda: G.gspmm(g, phi, rho, **kw), a.reps)
                    nb = op_bytes("gspmm", phi, rho, n, m, shapes, d_out, 4)
                    rows.append(dict(kernel="gspmm", phi=phi.describe(), rho=rho,
                                     strategy="node_parallel", format="csc", num_nodes=n,
                                     num_edges=m, feat_size=dim, heads=1, repeats=a.reps,
                                     median_seconds=t, gflops=2 * m * dim / t / 1e9,
                                     peak_aux_bytes=0, graph=gname, gbps=nb / t / 1e9,
                                     roofline_frac=nb / t / 1e9 / peak))
                t = timeit(lambda: G.gsddmm(g, phi, **kw), a.reps)
                nb = op_bytes("gsddmm", phi, "-", n, m, shapes, d_out, 4)
                rows.append(dict(kernel="gsddmm", phi=phi.describe(), rho="-",
                                 strategy="edge_parallel", format="coo", num_nodes=n,
                                 num_edges=m, feat_size=dim, heads=1, repeats=a.reps,
                                 median_seconds=t, gflops=2 * m * dim / t / 1e9,
                                 peak_aux_bytes=0, graph=gname, gbps=nb / t / 1e9,
                                 roofline_frac=nb / t / 1e9 / peak))
            print(gname, dim, "done", flush=True)
            del X, Y, W
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    with open(a.out, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=COLUMNS)
        w.writeheader()
        for r in rows:
            w.writerow({k: (round(v, 6) if isinstance(v, float) else v) for k, v in r.items()})
    fr = np.array([r["roofline_frac"] for r in rows])
    print("cells", len(rows), "roofline_frac median %.3f min %.3f" % (np.median(fr), fr.min()))
    worst = sorted(rows, key=lambda r: r["roofline_frac"])[:15]
    for r in worst:
        print("  worst", r["graph"], r["kernel"], r["phi"], r["rho"], r["feat_size"],
              "%.3f ms %.0f GB/s frac %.3f" % (r["median_seconds"] * 1e3, r["gbps"], r["roofline_frac"]))


if __name__ == "__main__":
    main()
