"""Host-side logic on CPU: validation, graph indexes, caches, instrumentation.

No kernel runs here; the graph lives on the CPU device, where every kernel
entry point must refuse to run (there is no CPU fallback).
"""

import threading

import numpy as np
import pytest
import torch

import paper_1909_01315_b200 as G
from paper_1909_01315_b200 import accounting, kernels
from conftest import golden, golden_graph, to_np


def cpu_graph(n, edges):
    return G.build_graph(n, edges, device="cpu")


def test_message_func_validation():
    with pytest.raises(ValueError):
        kernels.MessageFunc("mul", "src", "src")
    with pytest.raises(ValueError):
        kernels.MessageFunc("copy_lhs", "src", "dst")
    with pytest.raises(ValueError):
        kernels.MessageFunc("hypot", "src", "dst")
    phis = kernels.builtin_message_funcs()
    assert len(phis) == 30
    assert phis[0].describe() == "copy_lhs(src)"
    assert [p.describe() for p in phis[-3:]] == ["dot(src,dst)", "dot(src,edge)", "dot(dst,edge)"]


def test_graph_validation_errors():
    with pytest.raises(ValueError, match="outside"):
        G.Graph(np.array([0, 5]), np.array([1, 1]), 3, device="cpu")
    with pytest.raises(ValueError, match="negative"):
        G.build_graph(3, [(0, -1)], device="cpu")
    with pytest.raises(ValueError):
        G.Graph(np.array([0, 1]), np.array([1]), 3, device="cpu")


def test_adjacency_bit_exact_vs_reference():
    gd = golden()
    src, dst, n = golden_graph("idx")
    g = G.from_arrays(src, dst, num_nodes=n, device="cpu")
    for nm, adj in (("csc", g.to_csc()), ("csr", g.to_csr())):
        indptr, indices, eids = adj.numpy()
        assert np.array_equal(indptr, gd["idx/%s/indptr" % nm])
        assert np.array_equal(indices, gd["idx/%s/indices" % nm])
        assert np.array_equal(eids, gd["idx/%s/edge_ids" % nm])


def test_reverse_shares_cache_pair():
    g = cpu_graph(3, [(0, 2), (1, 2), (2, 0)])
    rev = G.reverse(g)
    assert G.reverse(rev) is g
    assert rev.to_csc() is g.to_csr()
    assert rev.to_csr() is g.to_csc()
    assert g.adjacency_build_count == 2
    rev.to_csc()
    assert g.adjacency_build_count == 2
    assert rev.uid != g.uid


def test_concurrent_cache_build_is_single():
    rng = np.random.default_rng(0)
    g = G.from_arrays(rng.integers(0, 50, 500), rng.integers(0, 50, 500), 50, device="cpu")
    barrier = threading.Barrier(8)
    got = []

    def run():
        barrier.wait()
        got.append(g.to_csc())

    ts = [threading.Thread(target=run) for _ in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert all(a is got[0] for a in got)
    assert g.adjacency_build_count == 1


def test_degrees():
    g = cpu_graph(3, [(0, 2), (1, 2), (2, 0)])
    assert to_np(g.in_degrees()).tolist() == [1, 0, 2]
    assert to_np(g.out_degrees()).tolist() == [1, 1, 1]
    g.to_csc()
    assert to_np(g.in_degrees([2, 0])).tolist() == [2, 1]
    with pytest.raises(IndexError):
        g.in_degrees([3])


def test_kernels_refuse_cpu_graph():
    g = cpu_graph(3, [(0, 2), (1, 2), (2, 0)])
    x = np.ones((3, 1))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        G.gspmm(g, kernels.copy("src"), "sum", X=x)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        G.gsddmm(g, kernels.copy("src"), X=x)


def test_validation_happens_before_device_check():
    g = cpu_graph(3, [(0, 2), (1, 2), (2, 0)])
    with pytest.raises(ValueError):
        G.gspmm(g, kernels.add("src", "dst"), "sum", X=np.ones((3, 2)), Y=np.ones((3, 3)))
    with pytest.raises(ValueError):
        G.gspmm(g, kernels.mul("src", "edge"), "sum", X=np.ones((3, 1)))
    with pytest.raises(ValueError):
        G.gspmm(g, kernels.copy("src"), "sum", X=np.ones((4, 1)))
    with pytest.raises(ValueError):
        G.gsddmm(g, kernels.copy_rhs("edge"), W=np.ones((2, 1)))
    with pytest.raises(ValueError):
        G.gsddmm(g, kernels.dot("src", "dst"), X=np.ones((3, 2)), Y=np.ones((3, 3)))
    with pytest.raises(ValueError):
        G.gspmm(g, kernels.copy("src"), "sum", X=np.ones((3, 1)), strategy="warp")
    with pytest.raises(ValueError):
        G.gspmm(g, kernels.copy("src"), "median", X=np.ones((3, 1)))
    with pytest.raises(ValueError, match="atomic"):
        G.gsddmm(g, kernels.copy("src"), X=np.ones((3, 1)), strategy="edge_parallel_atomic")
    with pytest.raises(ValueError):
        G.gspmm(g, kernels.copy("src"), "sum", X=np.ones((3, 1)), strategy="node_parallel",
                fmt="coo")
    with pytest.raises(ValueError):
        G.gspmm(g, kernels.copy("src"), "sum", X=np.ones((3,)))


def test_select_format():
    assert G.select_format("gspmm", "forward") == "csc"
    assert G.select_format("gspmm", "backward") == "csc"
    assert G.select_format("gsddmm") == "coo"
    with pytest.raises(ValueError):
        G.select_format("spmv")


def test_allocation_meter_and_dispatch_log(tmp_path):
    with pytest.raises(G.MemoryCapExceeded):
        with accounting.track_allocations(cap_bytes=100):
            accounting.register_bytes(101)
    with accounting.track_allocations() as meter:
        accounting.register(torch.zeros(10, 4))
        accounting.release_bytes(80)
    assert meter.peak_bytes == 160 and meter.current_bytes == 80
    assert meter.largest_single_bytes == 160
    with G.capture_dispatch() as log:
        accounting.log_dispatch("gspmm", 7, "copy_lhs(src)", "sum", "node_parallel", 3, 2)
    path = tmp_path / "d.log"
    accounting.write_dispatch_log(path, log)
    assert path.read_text().strip() == "gspmm,7,copy_lhs(src),sum,node_parallel,3,2"


def test_feature_dict():
    fd = G.FeatureDict(3, device="cpu")
    fd["h"] = np.array([1.0, 2.0, 3.0])
    assert tuple(fd["h"].shape) == (3, 1)
    assert "h" in fd and len(fd) == 1
    with pytest.raises(ValueError):
        fd["x"] = np.ones((4, 1))
    with pytest.raises(ValueError):
        fd["x"] = np.array([1.0, np.inf, 0.0])
    with pytest.raises(KeyError, match="have: h"):
        fd["nope"]
    with pytest.raises(ValueError):
        fd[""] = np.ones((3, 1))
    del fd["h"]
    assert len(fd) == 0


def test_messaging_host_errors():
    g = cpu_graph(3, [(0, 2), (1, 2), (2, 0)])
    nd = G.FeatureDict(3, device="cpu")
    nd["h"] = np.ones((3, 1))
    with pytest.raises(ValueError, match="edata"):
        G.apply_edges(g, G.msg("copy", G.src("h")), nd, out="m")
    with pytest.raises(ValueError, match="edata"):
        G.edge_softmax(g, "s")
    m = G.msg("copy_rhs", G.edge("w"))
    assert m.lhs is None and m.rhs.name == "w"


def test_generators_match_reference():
    gd = golden()
    g = G.power_law(400, 6, seed=3, device="cpu")
    assert np.array_equal(to_np(g.src), gd["gen/power_law_400_6_3/src"])
    assert np.array_equal(to_np(g.dst), gd["gen/power_law_400_6_3/dst"])
    spec = G.generators.parse_graph_spec("power_law:n=100,deg=3,seed=4")
    assert spec == G.GenSpec("power_law", 100, 3.0, 4)
    with pytest.raises(ValueError):
        G.generators.parse_graph_spec("chain:deg=3")


def test_rmat_cpu_shape_and_range():
    s, d = G.generators.rmat_edges(1000, 5000, seed=1, device="cpu")
    assert s.numel() == 5000 and int(s.max()) < 1000 and int(d.max()) < 1000
    s2, _ = G.generators.rmat_edges(1000, 5000, seed=1, device="cpu")
    assert torch.equal(s, s2)


# ---- round-1 additions: tiled path selection, window eid order, new APIs --

def test_tiled_path_selection():
    from paper_1909_01315_b200.kernels import _tiled_applies
    n = 232965
    X = torch.empty((n, 602))
    W = torch.empty((10, 1))
    cp = kernels.copy("src")
    assert _tiled_applies(cp, "sum", X, None, 602, n, None)
    assert _tiled_applies(cp, "mean", X, None, 602, n, None)
    assert not _tiled_applies(cp, "max", X, None, 602, n, None)      # arg output: untiled
    assert not _tiled_applies(cp, "sum", X[:, :64], None, 64, n, None)  # one tile
    assert not _tiled_applies(cp, "sum", torch.empty((n, 640)), None, 640, n, None)  # aligned
    assert not _tiled_applies(cp, "sum", X, None, 602, n, (62, 0))     # user tile override
    assert not _tiled_applies(cp, "sum", torch.empty((100, 602)), None, 602, 100, None)  # fits L2
    mul = kernels.mul("src", "edge")
    assert _tiled_applies(mul, "sum", X, W, 602, n, None)
    assert not _tiled_applies(mul, "sum", X, torch.empty((10, 602)), 602, n, None)
    assert not _tiled_applies(kernels.mul("dst", "edge"), "sum", X, W, 602, n, None)


def test_host_pipeline_tile_bounds():
    from paper_1909_01315_b200.pipeline import tile_bounds
    tiles, w = tile_bounds(602, 4)
    assert w == 64 and len(tiles) == 10
    assert tiles[0] == (0, 64) and tiles[-1] == (576, 602)
    tiles, w = tile_bounds(602, 8)
    assert w == 32 and tiles[-1] == (576, 602)


def test_sorted_eids_per_row_on_cpu():
    """_sorted_eids: the edge ids themselves when they ascend inside every
    CSC row, else a per-row sorted copy (torch ops only)."""
    g = cpu_graph(4, [(0, 1), (2, 1), (1, 0), (3, 1)])
    adj = g.to_csc()
    assert kernels._sorted_eids(adj) is adj.edge_ids
    # row 1 in CSC order: src 0 (e2), src 2 (e0), src 3 (e1) -> eids 2, 0, 1
    g2 = cpu_graph(4, [(2, 1), (3, 1), (0, 1), (1, 0)])
    a2 = g2.to_csc()
    se = kernels._sorted_eids(a2)
    assert se is not a2.edge_ids
    ip = to_np(a2.indptr)
    for r in range(4):
        seg = to_np(se)[ip[r]:ip[r + 1]]
        assert list(seg) == sorted(to_np(a2.edge_ids)[ip[r]:ip[r + 1]])


def test_new_entry_points_refuse_cpu_graph():
    g = cpu_graph(3, [(0, 2), (1, 2), (2, 0)])
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        G.neighbor_sample(g, [2], fanout=1, rng_seed=0)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        G.update_all_udf(g, lambda c: c.src_rows, lambda b: b.sum(dim=1),
                         src_feat=np.ones((3, 1)))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        kernels.edge_softmax_uv_stats(g, torch.zeros((3, 1)), torch.zeros((3, 1)))


def test_neighbor_sample_validates_before_device():
    g = cpu_graph(3, [(0, 2), (1, 2), (2, 0)])
    with pytest.raises(ValueError, match="fanout"):
        G.neighbor_sample(g, [0], fanout=0, rng_seed=0)
    with pytest.raises(IndexError):
        G.neighbor_sample(g, [7], fanout=2, rng_seed=0)


def test_layer_order_validation():
    from paper_1909_01315_b200 import layers
    W = torch.zeros((602, 16))
    assert layers._project_first(None, W, "auto")
    assert not layers._project_first(None, torch.zeros((16, 41)), "auto")
    assert layers._project_first(None, torch.zeros((16, 41)), "project_first")
    assert not layers._project_first(None, W, "aggregate_first")
    with pytest.raises(ValueError):
        layers._project_first(None, W, "sideways")


def test_tiled_path_sized_by_source_rows():
    """A row block of a partitioned graph gathers more source rows than it
    has destination rows: the L2 test and the packing use X's rows (ADVICE
    r1: the tiles were packed with the destination count)."""
    from paper_1909_01315_b200.kernels import _tiled_applies
    cp = kernels.copy("src")
    X = torch.empty((232965, 602))
    assert _tiled_applies(cp, "sum", X, None, 602, 2000, None)     # few destination rows
    assert not _tiled_applies(cp, "sum", torch.empty((2000, 602)), None, 602, 232965, None)


def test_models_know_their_output_width():
    from paper_1909_01315_b200 import layers
    m = layers.GATModel([12, 8, 8, 5], heads=2, seed=0, device="cpu")
    assert m.out_dim == 5
    assert layers.GCNModel([12, 8, 3], seed=0, device="cpu").out_dim == 3
    with pytest.raises(ValueError, match="divisible"):
        layers.GATModel([12, 9, 5], heads=2, seed=0, device="cpu")


def test_dense_precision_context():
    from paper_1909_01315_b200 import layers
    a = torch.randn(5, 7)
    b = torch.randn(7, 3)
    with layers.dense_precision("fp64"):
        got = layers._mm(a, b)
    assert got.dtype == torch.float32
    assert torch.equal(got, (a.double() @ b.double()).float())
    assert torch.equal(layers._mm(a, b), a @ b)
    with pytest.raises(ValueError):
        with layers.dense_precision("fp16"):
            pass
