"""Benchmark: g-SpMM achieved GB/s on the Reddit-shaped graph (BASELINE.json).

Workload (config C3, BASELINE.json configs[2]): the reference's own
power_law(232965, 492, seed=0) graph (m = 114,497,502), X ~ N(0,1) fp32 with
d = 602, one copy_u + sum g-SpMM per step (the first GCN layer's
aggregation). value = algorithmic bytes / kernel time with inputs resident in
HBM, bytes = (n+1)*8 + m*4 + m*d*4 + n*d*4. L2 is flushed
(256 MiB write) between timed steps, outside the timed events.

e2e: the same op through the public API (paper_1909_01315_b200.gspmm) with
X copied from pinned host memory before and Z copied back after, every step.
Extras: other ops of the sweep, fused edge_softmax, GCN / SAGE epoch ms.

N > 1 (torchrun): destination rows partitioned by equal edge counts; every
step all-gathers the row-sharded X over NCCL and runs the local rows
(strong scaling: the whole graph is fixed). Timing is max over ranks.

--impl reference: the CPU oracle port of the reference (oracle/gmp_oracle.py,
node_parallel restatement) on a bounded row sample, all host threads.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_NODES, AVG_DEG, FEAT, HIDDEN, CLASSES = 232_965, 492, 602, 16, 41


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--nodes", type=int, default=N_NODES)
    p.add_argument("--deg", type=int, default=AVG_DEG)
    p.add_argument("--feat", type=int, default=FEAT)
    p.add_argument("--no-extras", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-edges", type=int, default=24_000_000,
                   help="edges in the CPU baseline sample (strided rows)")
    p.add_argument("--tile-cols", type=int, default=0)
    p.add_argument("--workload", default="reddit", choices=["reddit", "rmat"],
                   help="reddit: config C3 (default); rmat: config C4, 10M nodes / 1B edges / d=256")
    a = p.parse_args()
    if a.workload == "rmat":
        a.nodes, a.edges = 10_000_000, 1_000_000_000
        if a.feat == FEAT:
            a.feat = 256
    return a


def spmm_bytes(n, m, d):
    return (n + 1) * 8 + m * 4 + m * d * 4 + n * d * 4


def peaks():
    path = ROOT / "MEASURED_PEAKS.json"
    if path.exists():
        try:
            return float(json.loads(path.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap,utilization.gpu",
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[2:6], float(parts[6])))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        loaded = [r for r in rows if r[3] > 0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[2])
                          if v.lower() == "active"})
        return {"sm_mhz": float(np.median([r[0] for r in loaded])),
                "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows), "samples_under_load": len(loaded)}


def build_graph_arrays(args):
    from paper_1909_01315_b200 import generators
    t0 = time.time()
    s, d = generators.power_law_edges(args.nodes, args.deg, seed=0)
    return s, d, time.time() - t0


# ----------------------------------------------------------------- CPU leg ---

def strided_rows(indptr, n_edges_target):
    """Every k-th destination row of the CSC, k chosen so the sample holds
    ~n_edges_target edges: a cross-section of the whole degree distribution
    (hubs and the long tail), not a prefix of hub rows."""
    n = indptr.size - 1
    m = int(indptr[-1])
    k = max(1, int(round(m / max(1, n_edges_target))))
    return np.arange(0, n, k, dtype=np.int64)


def sub_csc(indptr, indices, eids, rows):
    lens = (indptr[rows + 1] - indptr[rows]).astype(np.int64)
    sub_ptr = np.zeros(rows.size + 1, dtype=np.int64)
    np.cumsum(lens, out=sub_ptr[1:])
    pos = np.repeat(indptr[rows] - sub_ptr[:-1], lens) + np.arange(int(sub_ptr[-1]), dtype=np.int64)
    return sub_ptr, indices[pos], eids[pos]


def cpu_sample(indptr, indices, eids, x, n_edges_target, workers):
    """Time the oracle's node_parallel g-SpMM (the reference algorithm,
    kernels.py:473-482) on a strided sample of destination rows holding
    ~n_edges_target edges. Returns (seconds, algorithmic bytes, rows, edges)."""
    from oracle import gmp_oracle as O
    rows = strided_rows(indptr, n_edges_target)
    sub_ptr, sub_ind, sub_eid = sub_csc(indptr, indices, eids, rows)
    # only the source rows the sample touches are handed to the CPU (the
    # gathers read the same values; keeps host memory bounded on 1B edges)
    used, remap = np.unique(sub_ind, return_inverse=True)
    x = np.asarray(x[used], dtype=np.float64)
    sub = (sub_ptr, remap.astype(np.int64), sub_eid)
    r, e = rows.size, int(sub_ptr[-1])
    d = x.shape[1]
    t0 = time.perf_counter()
    O.gspmm(None, None, r, "copy_lhs", "src", None, "sum", X=x, workers=workers, adj=sub)
    dt = time.perf_counter() - t0
    return dt, spmm_bytes(r, e, d), r, e


def run_reference(args):
    """--impl reference: the CPU port of the reference's node_parallel g-SpMM."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import gmp_oracle as O
    s, d, gen_s = build_graph_arrays(args)
    n, m = args.nodes, s.size
    # CSC with the reference's ordering (graph.py:35-44), built by one stable
    # argsort of dst * n + src (equivalent to its lexsort; not timed)
    order = np.argsort(d.astype(np.int64) * n + s, kind="stable")
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(d, minlength=n), out=indptr[1:])
    indices, eids = s[order], order
    rng = np.random.default_rng(0)
    x = rng.standard_normal((n, args.feat), dtype=np.float32).astype(np.float64)
    workers = len(os.sched_getaffinity(0))
    sample_edges = min(args.cpu_edges // 4, m)
    for _ in range(args.warmup):
        cpu_sample(indptr, indices, eids, x, max(1, sample_edges // 20), workers)
    secs, nbytes = 0.0, 0
    for _ in range(args.steps):
        dt, b, r, e = cpu_sample(indptr, indices, eids, x, sample_edges, workers)
        secs += dt
        nbytes += b
    gbs = nbytes / secs / 1e9
    line = {
        "impl": "reference", "metric": "g-SpMM achieved GB/s (copy_u+sum, Reddit-shaped, d=%d)" % args.feat,
        "value": round(gbs, 3), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(secs / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference power_law(%d, %d, seed=0) graph, X~N(0,1)" % (n, args.deg),
        "config": {"workload": "reddit_spmm_copy_u_sum", "nodes": n, "edges": int(m),
                   "feat": args.feat, "sample_rows": r, "sample_edges": e},
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": workers, "kind": "port",
                         "sample": "every k-th CSC row: %d rows / %d edges of the Reddit-shaped "
                                   "graph per step, d=%d" % (r, e, args.feat)},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU leg ---

def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_1909_01315_b200 as G
    from paper_1909_01315_b200 import _lib, distributed, kernels, layers

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # GMP_BENCH_BACKEND=gloo lets the N>1 path be smoke-tested with several
        # ranks on one GPU; the measured configuration is NCCL, one rank per GPU
        backend = os.environ.get("GMP_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    torch.backends.cuda.matmul.allow_tf32 = False

    if args.workload == "rmat":
        t0 = time.time()
        g = G.rmat(args.nodes, args.edges, seed=0, device=dev)
        torch.cuda.synchronize()
        gen_s = time.time() - t0
    else:
        s, d, gen_s = build_graph_arrays(args)
    n, m, F = args.nodes, (int(args.edges) if args.workload == "rmat" else int(s.size)), args.feat
    t0 = time.time()
    if args.workload != "rmat":
        g = G.from_arrays(s, d, num_nodes=n, device=dev)
    adj = g.to_csc()
    adj.schedule()
    torch.cuda.synchronize()
    build_s = time.time() - t0
    gen = torch.Generator(device=dev)
    gen.manual_seed(0)
    X = torch.randn((n, F), generator=gen, device=dev, dtype=torch.float32)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    phi = kernels.copy("src")
    tune = None
    if args.tile_cols:
        tune = kernels.tuning(tile_cols=args.tile_cols)
        tune.__enter__()

    if world > 1:
        pg = distributed.PartitionedGraph(adj, n, rank, world)
        x_local = X[pg.r0:pg.r1].contiguous()
        for blk in (pg.block, pg.local_block, pg.remote_block):
            blk.to_csc().schedule()

        def step():
            return pg.aggregate(x_local, "sum", overlap=True)
        step_bytes = spmm_bytes(n, m, F)
    else:
        def step():
            return G.gspmm(g, phi, "sum", X=X)[0]
        step_bytes = spmm_bytes(n, m, F)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream(dev)
    launches0 = _lib.launch_count()
    times = []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step()
            b.record(stream)
            b.synchronize()
            times.append(a.elapsed_time(b))
    torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    ms = float(np.mean(times))
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    value = step_bytes / (ms * 1e-3) / 1e9
    peak, peak_kind = peaks()

    # e2e through the public API with host buffers: pipeline.gspmm_host takes
    # pinned host X and returns host Z, H2D / kernel / D2H overlapped per tile
    e2e = None
    if world == 1:
        from paper_1909_01315_b200 import pipeline
        xh = X.cpu().pin_memory()
        zh = torch.empty((n, F), dtype=torch.float32).pin_memory()
        pipe = pipeline.HostPipeline(dev)
        e2e_times = []
        for i in range(args.warmup + args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            pipeline.gspmm_host(g, xh, zh, "sum", pipe=pipe)
            b.record(stream)
            b.synchronize()
            if i >= args.warmup:
                e2e_times.append(a.elapsed_time(b))
        e2e_ms = float(np.mean(e2e_times))
        e2e = {"value": round(step_bytes / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
               "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": int(xh.numel() * 4),
               "d2h_bytes_per_step": int(zh.numel() * 4),
               "api": "paper_1909_01315_b200.pipeline.gspmm_host (pinned host X -> host Z, "
                      "copies overlapped with the kernel per column tile)"}
        zref = G.gspmm(g, phi, "sum", X=X)[0].cpu()
        e2e["matches_device_result"] = bool(torch.equal(zref, zh))

    extras = {}
    if rank == 0 and world == 1 and not args.no_extras:
        extras = run_extras(G, kernels, layers, g, X, n, m, flush, stream, dev, args)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        indptr, indices, eids = adj.numpy()
        workers = len(os.sched_getaffinity(0))
        xc = X.cpu().numpy()
        dt, nb, r, e = cpu_sample(indptr, indices.astype(np.int64), eids.astype(np.int64), xc,
                                  args.cpu_edges, workers)
        cpu = {"value": round(nb / dt / 1e9, 3), "unit": "GB/s", "cores": workers, "kind": "port",
               "seconds": round(dt, 2),
               "sample": "oracle node_parallel copy_u+sum on every k-th CSC row: %d rows / %d "
                         "edges, d=%d, %d threads" % (r, e, F, workers)}

    traffic = None
    l2 = None
    tpath = ROOT / "profiles" / "ncu_traffic.json"
    if tpath.exists():
        try:
            tj = json.loads(tpath.read_text())
            if tj.get("feat") == F and tj.get("edges") == m:
                traffic = tj.get("dram_bytes_per_launch")
                l2b = tj.get("row_kernel_l2_read_bytes")
                cpath = ROOT / "profiles" / "l2_gather_ceiling.json"
                if l2b and cpath.exists():
                    ceil = float(json.loads(cpath.read_text())["ceiling_gbs_60mb"])
                    ach = l2b / (ms * 1e-3) / 1e9
                    l2 = {"read_bytes_per_step": l2b, "achieved_gbs": round(ach, 1),
                          "gather_ceiling_gbs": ceil, "frac": round(ach / ceil, 4),
                          "source": "profiles/ncu_traffic.json (ncu L2 sectors of the row "
                                    "kernel launches) over this run's step time; ceiling "
                                    "profiles/l2_gather_ceiling.json"}
        except Exception:
            traffic = None

    if rank == 0:
        sched = adj.schedule()
        line = {
            "metric": "g-SpMM achieved GB/s (copy_u+sum, %s, d=%d)" % (
                "Reddit-shaped" if args.workload == "reddit" else "RMAT 10M/1B", F),
            "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 (fp64 accumulate)",
            "data": ("synthetic: reference power_law(%d, %d, seed=0) graph, X~N(0,1)" % (n, args.deg)
                     if args.workload == "reddit" else
                     "synthetic: Graph500 R-MAT (0.57,0.19,0.19) on device, seed 0, X~N(0,1)"),
            "config": {"workload": ("reddit" if args.workload == "reddit" else "rmat")
                       + "_spmm_copy_u_sum", "nodes": n, "edges": m, "feat": F,
                       "heavy_rows": sched.n_heavy, "nonempty_rows": sched.n_nonempty,
                       "l2": "flushed between steps (256 MiB write, outside timed events)",
                       "parallelism": "row-partition x%d" % world if world > 1 else "single GPU",
                       "graph_gen_s": round(gen_s, 1), "csc_build_s": round(build_s, 2)},
            "roofline": {"bound": "hbm", "achieved": round(value, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(value / peak, 4), "traffic": traffic,
                         "peak_kind": peak_kind,
                         "kernel": "spmm_rows_kernel<float,COPY,SUM> over packed 256 B column tiles",
                         "bytes_per_launch": step_bytes,
                         "note": "achieved = algorithmic (no-reuse) bytes per step / step time; "
                                 "frac > 1 because each column tile of X is L2-resident while "
                                 "every row gathers it - traffic is the measured DRAM bytes and "
                                 "l2 the bound that binds",
                         "l2": l2},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks.summary(),
            "gpu_launches": int(launches),
            "extras": extras,
        }
        print(json.dumps(line), flush=True)
    if tune is not None:
        tune.__exit__(None, None, None)
    if world > 1:
        dist.destroy_process_group()


def _time(fn, stream, flush, reps=5):
    import torch
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def run_extras(G, kernels, layers, g, X, n, m, flush, stream, dev, args):
    import torch
    out = {}
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    F = X.shape[1]
    w1 = torch.randn((m, 1), generator=gen, device=dev)
    x16 = torch.randn((n, 16), generator=gen, device=dev)
    cases = [
        ("copy_u_sum_d16", lambda: G.gspmm(g, kernels.copy("src"), "sum", X=x16),
         spmm_bytes(n, m, 16)),
        ("copy_u_max_d16", lambda: G.gspmm(g, kernels.copy("src"), "max", X=x16),
         spmm_bytes(n, m, 16) + n * 16 * 8),
        ("u_mul_e_sum_d%d" % F, lambda: G.gspmm(g, kernels.mul("src", "edge"), "sum", X=X, W=w1),
         spmm_bytes(n, m, F) + m * 4 + m * 4),
        ("u_dot_v_d16", lambda: G.gsddmm(g, kernels.dot("src", "dst"), X=x16, Y=x16),
         2 * m * 4 + 2 * m * 16 * 4 + m * 4),
    ]
    s8 = torch.randn((m, 8), generator=gen, device=dev)
    cases.append(("edge_softmax_h8", lambda: G.edge_softmax(g, s8),
                  (n + 1) * 8 + m * 4 + 2 * m * 8 * 4))
    for name, fn, nbytes in cases:
        t = _time(fn, stream, flush)
        out[name] = {"ms": round(t, 4), "GB/s": round(nbytes / (t * 1e-3) / 1e9, 1)}
    labels = torch.randint(0, CLASSES, (n,), generator=gen, device=dev)
    gcn = layers.GCNModel([F, HIDDEN, CLASSES], seed=0, device=dev)
    out["gcn_epoch_ms"] = round(_time(lambda: layers.train_epoch(g, X, labels, gcn, 0.01),
                                      stream, flush, reps=3), 3)
    gcn_af = layers.GCNModel([F, HIDDEN, CLASSES], seed=0, device=dev, order="aggregate_first")
    out["gcn_epoch_aggregate_first_ms"] = round(
        _time(lambda: layers.train_epoch(g, X, labels, gcn_af, 0.01), stream, flush, reps=3), 3)
    sage = layers.SAGEModel([F, HIDDEN, CLASSES], seed=0, device=dev)
    out["sage_epoch_ms"] = round(_time(lambda: layers.train_epoch(g, X, labels, sage, 0.01),
                                       stream, flush, reps=3), 3)
    gat = layers.GATModel([F, HIDDEN, HIDDEN, CLASSES], heads=1, seed=0, device=dev)
    out["gat_epoch_ms"] = round(_time(lambda: layers.train_epoch(g, X, labels, gat, 0.01),
                                      stream, flush, reps=3), 3)
    return out


if __name__ == "__main__":
    main()
