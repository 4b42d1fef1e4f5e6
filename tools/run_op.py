"""Run one hot-path op on the Reddit-shaped graph (for ncu / quick timing).

    python tools/run_op.py --op copy_sum --feat 602 --reps 3 [--time]
ops: copy_sum copy_max umul_sum umul_full_sum softmax softmax_bwd dot_sddmm add_sddmm gcn_epoch
"""

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_1909_01315_b200 as G  # noqa: E402
from paper_1909_01315_b200 import kernels, layers  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--op", default="copy_sum")
    p.add_argument("--feat", type=int, default=602)
    p.add_argument("--nodes", type=int, default=232965)
    p.add_argument("--deg", type=int, default=492)
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=2)
    p.add_argument("--time", action="store_true")
    p.add_argument("--tile-cols", type=int, default=0)
    p.add_argument("--l2mb", type=int, default=0)
    p.add_argument("--rmat", type=int, default=0, help="RMAT edge count (nodes = --nodes)")
    p.add_argument("--edge-cache", default="", help="npz file caching the power_law edges")
    p.add_argument("--l2fetch", type=int, default=0, help="cudaLimitMaxL2FetchGranularity bytes")
    p.add_argument("--profile", action="store_true",
                   help="cudaProfilerStart/Stop around the timed reps (ncu --profile-from-start off)")
    a = p.parse_args()
    dev = torch.device("cuda")
    torch.zeros(1, device=dev)
    if a.l2fetch:
        import ctypes
        rt = ctypes.CDLL("libcudart.so.12")
        v = ctypes.c_size_t(0)
        rc = rt.cudaDeviceSetLimit(5, ctypes.c_size_t(a.l2fetch))
        rt.cudaDeviceGetLimit(ctypes.byref(v), 5)
        print("l2 fetch granularity set rc=%d now %d" % (rc, v.value))
    import time
    t0 = time.time()
    if a.rmat:
        n = a.nodes
        g = G.rmat(n, a.rmat, seed=0, device=dev)
        m, F = g.num_edges, a.feat
    else:
        if a.edge_cache and Path(a.edge_cache).exists():
            z = np.load(a.edge_cache)
            s, d = z["s"], z["d"]
        else:
            s, d = G.generators.power_law_edges(a.nodes, a.deg, seed=0)
            if a.edge_cache:
                np.savez(a.edge_cache, s=s, d=d)
        n, m, F = a.nodes, s.size, a.feat
        g = G.from_arrays(s, d, num_nodes=n, device=dev)
    torch.cuda.synchronize()
    t1 = time.time()
    g.to_csc().schedule()
    torch.cuda.synchronize()
    if a.time:
        print("graph: n=%d m=%d gen %.1fs csc+schedule %.1fs heavy=%d" % (
            n, m, t1 - t0, time.time() - t1, g.to_csc().schedule().n_heavy))
    gen = torch.Generator(device=dev)
    gen.manual_seed(0)
    X = torch.randn((n, F), generator=gen, device=dev)
    W1 = torch.randn((m, 1), generator=gen, device=dev) if a.op.startswith("umul") else None
    ops = {
        "copy_sum": lambda: G.gspmm(g, kernels.copy("src"), "sum", X=X),
        "copy_max": lambda: G.gspmm(g, kernels.copy("src"), "max", X=X),
        "umul_sum": lambda: G.gspmm(g, kernels.mul("src", "edge"), "sum", X=X, W=W1),
        "dot_sddmm": lambda: G.gsddmm(g, kernels.dot("src", "dst"), X=X, Y=X),
        "add_sddmm": lambda: G.gsddmm(g, kernels.add("src", "dst"), X=X, Y=X),
    }
    if a.op in ("softmax", "softmax_bwd"):
        S = torch.randn((m, F), generator=gen, device=dev)
        alpha = G.edge_softmax(g, S)
        ops["softmax"] = lambda: G.edge_softmax(g, S)
        ops["softmax_bwd"] = lambda: kernels.edge_softmax_backward(g, alpha, S)
    if a.op == "umul_full_sum":
        WF = torch.randn((m, F), generator=gen, device=dev)
        ops["umul_full_sum"] = lambda: G.gspmm(g, kernels.mul("src", "edge"), "sum", X=X, W=WF)
    if a.op == "gcn_epoch":
        labels = torch.randint(0, 41, (n,), generator=gen, device=dev)
        model = layers.GCNModel([F, 16, 41], seed=0, device=dev)
        ops["gcn_epoch"] = lambda: layers.train_epoch(g, X, labels, model, 0.01)
    if a.op == "gat_epoch":
        labels = torch.randint(0, 41, (n,), generator=gen, device=dev)
        model = layers.GATModel([F, 16, 16, 41], heads=1, seed=0, device=dev)
        ops["gat_epoch"] = lambda: layers.train_epoch(g, X, labels, model, 0.01)
    fn = ops[a.op]
    ctx = kernels.tuning(tile_cols=a.tile_cols or None, l2_budget_mb=a.l2mb or None)
    with ctx:
        for _ in range(a.warmup):
            fn()
        torch.cuda.synchronize()
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        ts = []
        if a.profile:
            torch.cuda.profiler.start()
        for _ in range(a.reps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        if a.profile:
            torch.cuda.profiler.stop()
    if a.time:
        print("%s feat=%d tile=%d l2mb=%d: median %.3f ms (all %s)" % (
            a.op, F, a.tile_cols, a.l2mb, float(np.median(ts)), [round(t, 3) for t in ts]))


if __name__ == "__main__":
    main()
