"""Op sweep (BASELINE.json config C5): every built-in phi x rho
for g-SpMM and every phi for g-SDDMM, feature dims 1..512, on the reference's
uniform graph constant_indegree(n, 32, 0) and power-law graph power_law(n, 20,
0) (/root/reference/pkg/src/graphmp/generators.py:52-96), beside the
reference CPU path.

CSV: the reference bench schema (bench.py:39-41 COLUMNS: kernel, phi, rho,
strategy, format, num_nodes, num_edges, feat_size, heads, repeats,
median_seconds, gflops, peak_aux_bytes) extended with
  graph, gbps, roofline_frac     algorithmic bytes / median time,
                                 fraction of MEASURED_PEAKS hbm_gbs
  cpu_seconds, cpu_gbps,         the reference (graphmp from baseline/_ref;
  cpu_cores, cpu_kind, cpu_sample  the oracle port if absent) on a bounded
                                 sample of the same cell: every k-th destination
                                 row with all its in-edges (g-SpMM) / every k-th
                                 edge (g-SDDMM), ~4M message elements, default
                                 strategy, all host cores, one call after a
                                 warm-up call
  parity, parity_max_abs         the GPU result on the sample's rows / edges
                                 against that reference call: max/min values
                                 and arg edges bit-exact (dot: tolerance),
                                 sum/mean/elementwise rtol 1e-5 / atol 1e-6
  ncu_dram_gbps, ncu_dram_over_alg  filled by --merge-ncu from an ncu launch
                                 list of a --ncu-pass run (dram__bytes_read +
                                 write of the cell's launches / their duration)
gflops uses the reference's continuity formula 2 * m * d (bench.py:146).
Operands of div are |N(0,1)| + 0.5 (conftest.py:37-39); all operands use it.

    python tools/op_sweep.py --nodes 1000000 --out gpurun_out/op_sweep.csv
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --csv --log-file gpurun_out/sweep_ncu.csv python tools/op_sweep.py --ncu-pass
    python tools/op_sweep.py --merge-ncu gpurun_out/sweep_ncu.csv --out gpurun_out/op_sweep.csv
"""

import argparse
import csv
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

COLUMNS = ("kernel", "phi", "rho", "strategy", "format", "num_nodes", "num_edges", "feat_size",
           "heads", "repeats", "median_seconds", "gflops", "peak_aux_bytes", "graph", "gbps",
           "roofline_frac", "cpu_seconds", "cpu_gbps", "cpu_cores", "cpu_kind", "cpu_sample",
           "parity", "parity_max_abs", "ncu_dram_gbps", "ncu_dram_over_alg")
RTOL, ATOL = 1e-5, 1e-6
CPU_ELEMS = 4_000_000


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


def timeit(torch, fn, reps):
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


def graph_edges(name, n):
    from paper_1909_01315_b200 import generators
    if name == "uniform":
        return generators.constant_indegree_edges(n, 32, seed=0)
    return generators.power_law_edges(n, 20, seed=0)


class RefCells:
    """The reference on bounded samples of a sweep cell."""

    def __init__(self):
        import bench
        self.bench = bench
        self.mod, self.kind = bench.load_reference()
        self.cores = len(os.sched_getaffinity(0))

    def phi(self, phi):
        K = self.mod.kernels if self.kind == "reference" else None
        if K is None:
            return phi
        return K.MessageFunc(phi.op, phi.lhs_target, phi.rhs_target)

    def graph(self, src, dst, n):
        if self.kind != "reference":
            return (src, dst, n)
        g = self.mod.from_arrays(src.astype(np.uint32), dst.astype(np.uint32), num_nodes=n)
        g.to_csc()
        return g

    def call(self, kind, g, phi, rho, ops):
        if self.kind == "reference":
            G = self.mod
            f = self.phi(phi)
            with G.kernels.default_workers(self.cores):
                if kind == "gspmm":
                    z, aux = G.gspmm(g, f, rho, **ops)
                    return z, (aux.arg_edge if rho in ("max", "min") else None)
                return G.gsddmm(g, f, **ops), None
        O = self.mod
        src, dst, n = g
        if kind == "gspmm":
            z, aux = O.gspmm(src, dst, n, phi.op, phi.lhs_target, phi.rhs_target, rho,
                             workers=self.cores, **ops)
            return z, (aux if rho in ("max", "min") else None)
        return O.gsddmm(src, dst, n, phi.op, phi.lhs_target, phi.rhs_target,
                        workers=self.cores, **ops), None

    def timed(self, kind, g, phi, rho, ops):
        self.call(kind, g, phi, rho, ops)  # warm-up (pool start-up, caches)
        t0 = time.perf_counter()
        out = self.call(kind, g, phi, rho, ops)
        return out, time.perf_counter() - t0


def cmp(got, want, exact):
    # the reference is fed the fp32 operands as fp64 arrays, so its output is
    # the fp64 message; for fp32 operands it returns that message rounded to
    # fp32 (the golden vectors), which is what the bit-exact bar compares
    dt = np.asarray(got).dtype
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    if exact:
        ok = got == want.astype(dt).astype(np.float64)
    else:
        ok = np.isclose(got, want, rtol=RTOL, atol=ATOL)
    diff = np.abs(got - want)
    return bool(ok.all()), float(diff.max()) if diff.size else 0.0


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--nodes", type=int, default=1_000_000)
    p.add_argument("--dims", default="1,2,4,8,16,32,64,128,256,512")
    p.add_argument("--graphs", default="uniform,power_law")
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--out", default="gpurun_out/op_sweep.csv")
    p.add_argument("--quick", action="store_true", help="one phi per op family")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--ncu-pass", action="store_true",
                   help="one launch per cell after a marker kernel, no timing (run under ncu)")
    p.add_argument("--merge-ncu", default="", help="ncu launch-list CSV of a --ncu-pass run")
    a = p.parse_args()
    if a.merge_ncu:
        merge_ncu(a)
        return

    import torch
    import paper_1909_01315_b200 as G
    from paper_1909_01315_b200 import kernels
    dev = torch.device("cuda")
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    n = a.nodes
    phis = kernels.builtin_message_funcs()
    if a.quick:
        keep = {"copy_lhs(src)", "copy_lhs(edge)", "mul(src,edge)", "add(src,dst)",
                "sub(edge,dst)", "div(src,edge)", "dot(src,dst)"}
        phis = [f for f in phis if f.describe() in keep]
    ref = None if (a.no_cpu or a.ncu_pass) else RefCells()
    rows, cells = [], []
    for gname in a.graphs.split(","):
        s, d = graph_edges(gname, n)
        g = G.from_arrays(s, d, num_nodes=n, device=dev)
        g.to_csc().schedule()
        m = g.num_edges
        if ref is not None:
            import bench
            indptr, indices, eids = bench.host_csc(s, d, n)
        for dim in [int(x) for x in a.dims.split(",")]:
            gen = torch.Generator(device=dev)
            gen.manual_seed(dim)
            X = torch.randn((n, dim), generator=gen, device=dev).abs() + 0.5  # div-safe
            Y = torch.randn((n, dim), generator=gen, device=dev).abs() + 0.5
            W = torch.randn((m, dim), generator=gen, device=dev).abs() + 0.5
            ops = {"src": ("X", X), "dst": ("Y", Y), "edge": ("W", W)}
            if ref is not None:
                target = max(4096, CPU_ELEMS // dim)
                rs = bench.RowSample(indptr, indices, eids, target)
                es = bench.EdgeSample(s, d, target)
                rows_t = torch.as_tensor(rs.rows, device=dev)
                geid_t = torch.as_tensor(es.geid, device=dev)
                Xh, Yh, Wh = X.cpu().numpy(), Y.cpu().numpy(), None
                wpos = torch.as_tensor(rs.geid, device=dev)
                r_ops = {"X": rs.pad(Xh[rs.used].astype(np.float64)),
                         "Y": np.zeros((rs.n, dim)), "W": W[wpos].cpu().numpy().astype(np.float64)}
                r_ops["Y"][:rs.rows.size] = Yh[rs.rows]
                e_ops = {"X": Xh[es.nodes].astype(np.float64), "Y": Yh[es.nodes].astype(np.float64),
                         "W": W[geid_t].cpu().numpy().astype(np.float64)}
                rg = ref.graph(rs.src, rs.dst, rs.n)
                eg = ref.graph(es.src, es.dst, es.n)
            for phi in phis:
                kw = {ops[t][0]: ops[t][1] for t in phi.targets}
                shapes = {t: dim for t in phi.targets}
                d_out = 1 if phi.op == "dot" else dim
                for kind, rho in [("gspmm", r) for r in ("sum", "mean", "max", "min")] + \
                        [("gsddmm", "-")]:
                    fn = (lambda: G.gspmm(g, phi, rho, **kw)) if kind == "gspmm" else \
                        (lambda: G.gsddmm(g, phi, **kw))
                    cell = dict(kernel=kind, phi=phi.describe(), rho=rho,
                                strategy="node_parallel" if kind == "gspmm" else "edge_parallel",
                                format="csc" if kind == "gspmm" else "coo", num_nodes=n,
                                num_edges=m, feat_size=dim, heads=1, graph=gname)
                    nb = op_bytes(kind, phi, rho, n, m, shapes, d_out, 4)
                    cell["_alg"] = nb
                    if a.ncu_pass:
                        torch.cuda._sleep(1000)  # marker kernel: cells are split on it
                        fn()
                        torch.cuda.synchronize()
                        cells.append(cell)
                        continue
                    t = timeit(torch, fn, a.reps)
                    cell.update(repeats=a.reps, median_seconds=t, gflops=2 * m * dim / t / 1e9,
                                peak_aux_bytes=0, gbps=nb / t / 1e9,
                                roofline_frac=nb / t / 1e9 / peak)
                    if ref is not None:
                        cell.update(ref_cell(ref, kind, phi, rho, fn, rs, es, rg, eg, r_ops,
                                             e_ops, rows_t, geid_t, dim, d_out))
                    rows.append(cell)
            print(gname, dim, "done", flush=True)
            del X, Y, W
            torch.cuda.empty_cache()
    if a.ncu_pass:
        Path(a.out).with_suffix(".cells.json").write_text(json.dumps(cells))
        return
    write(a.out, rows)
    summarise(rows)


def ref_cell(ref, kind, phi, rho, fn, rs, es, rg, eg, r_ops, e_ops, rows_t, geid_t, dim, d_out):
    """Reference time + parity of one cell on its bounded sample."""
    if kind == "gspmm":
        z, aux = fn()
        got = z[rows_t].cpu().numpy()
        garg = aux.arg_edge[rows_t].cpu().numpy() if rho in ("max", "min") else None
        kw = {k: r_ops[k] for k in ("X", "Y", "W") if any(
            {"src": "X", "dst": "Y", "edge": "W"}[t] == k for t in phi.targets)}
        (want, warg), secs = ref.timed(kind, rg, phi, rho, kw)
        want = np.asarray(want)[:rs.rows.size]
        smp_m, smp_n, smp = rs.m, rs.rows.size, rs.describe()
        exact = rho in ("max", "min") and phi.op != "dot"
        ok, mx = cmp(got, want, exact)
        if warg is not None and phi.op != "dot":
            warg = np.asarray(warg)[:rs.rows.size]
            warg = np.where(warg >= 0, rs.geid[np.maximum(warg, 0)], -1)
            ok = ok and bool(np.array_equal(garg, warg))
    else:
        mm = fn()
        got = mm[geid_t].cpu().numpy()
        kw = {k: e_ops[k] for k in ("X", "Y", "W") if any(
            {"src": "X", "dst": "Y", "edge": "W"}[t] == k for t in phi.targets)}
        (want, _), secs = ref.timed(kind, eg, phi, rho, kw)
        smp_m, smp_n, smp = es.m, es.n, es.describe()
        ok, mx = cmp(got, want, phi.op not in ("dot",))
    shapes = {t: dim for t in phi.targets}
    sb = op_bytes(kind, phi, rho, smp_n, smp_m, shapes, d_out, 4)
    return dict(cpu_seconds=secs, cpu_gbps=sb / secs / 1e9, cpu_cores=ref.cores,
                cpu_kind=ref.kind, cpu_sample=smp, parity="ok" if ok else "FAIL",
                parity_max_abs=mx)


def write(path, rows):
    Path(path).parent.mkdir(parents=True, exist_ok=True)
    with open(path, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=COLUMNS, extrasaction="ignore")
        w.writeheader()
        for r in rows:
            w.writerow({k: (float("%.6g" % v) if isinstance(v, float) else v) for k, v in r.items()})


def summarise(rows):
    fr = np.array([float(r["roofline_frac"]) for r in rows])
    print("cells", len(rows), "roofline_frac median %.3f min %.3f" % (np.median(fr), fr.min()))
    for k in ("gspmm", "gsddmm"):
        sub = np.array([float(r["roofline_frac"]) for r in rows if r["kernel"] == k])
        if sub.size:
            print("  %s median %.3f" % (k, np.median(sub)))
    bad = [r for r in rows if r.get("parity") == "FAIL"]
    print("parity: %d cells checked, %d FAIL" % (sum(1 for r in rows if r.get("parity")), len(bad)))
    for r in bad[:20]:
        print("  FAIL", r["graph"], r["kernel"], r["phi"], r["rho"], r["feat_size"],
              r["parity_max_abs"])
    worst = sorted(rows, key=lambda r: float(r["roofline_frac"]))[:15]
    for r in worst:
        print("  worst", r["graph"], r["kernel"], r["phi"], r["rho"], r["feat_size"],
              "%.3f ms %.0f GB/s frac %.3f" % (float(r["median_seconds"]) * 1e3,
                                               float(r["gbps"]), float(r["roofline_frac"])))


def merge_ncu(a):
    """Attach ncu DRAM GB/s to the sweep CSV: the launch list of a --ncu-pass
    run is split on its marker kernels, group k = cell k of the .cells.json."""
    cells = json.loads(Path(a.out).with_suffix(".cells.json").read_text())
    lines = [ln for ln in open(a.merge_ncu) if ln.startswith('"')]
    rd = list(csv.reader(lines))
    h = rd[0]
    ki, mi, vi, ui = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("Metric Unit"))
    idi = h.index("ID")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
             "usecond": 1e-6, "msecond": 1e-3, "second": 1}
    launches = {}
    for r in rd[1:]:
        L = launches.setdefault(int(r[idi]), {"name": r[ki]})
        L[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    groups, cur = [], None
    for i in sorted(launches):
        L = launches[i]
        if "spin" in L["name"] or "sleep" in L["name"]:
            cur = []
            groups.append(cur)
        elif cur is not None:
            cur.append(L)
    if len(groups) != len(cells):
        raise SystemExit("ncu groups %d != cells %d" % (len(groups), len(cells)))
    key = {}
    for c, grp in zip(cells, groups):
        byts = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in grp)
        t = sum(x.get("gpu__time_duration.sum", 0) for x in grp)
        key[(c["graph"], c["kernel"], c["phi"], c["rho"], str(c["feat_size"]))] = (
            byts / t / 1e9 if t else None, byts / c["_alg"])
    rows = list(csv.DictReader(open(a.out)))
    for r in rows:
        v = key.get((r["graph"], r["kernel"], r["phi"], r["rho"], r["feat_size"]))
        if v:
            r["ncu_dram_gbps"], r["ncu_dram_over_alg"] = v
    write(a.out, rows)
    print("merged", sum(1 for r in rows if r.get("ncu_dram_gbps")), "of", len(rows))


if __name__ == "__main__":
    main()
