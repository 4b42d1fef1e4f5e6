"""Pipelined gather ring of the row g-SpMM (spmm_accumulate_pipe,
spmm_rows.cuh): copy_u / u_mul_e + sum/mean over 64 / 128 / 256 B rows (4 /
8 / 16 lanes per edge; the fused GAT modes are covered by
test_gpu_gat_fused.py), heavy rows
(one CTA), medium rows (one warp) and light rows (two per warp) - against the
oracle at the fp32 bar, including a hub row whose exact sum cancels (a plain
fp32 accumulation misses the bar there by orders of magnitude), ragged last
batches, run-to-run determinism, and a subprocess with GMP_NO_PIPE=1 (the
burst kernel) for the heavy and medium rows, which keep the same edge order
and fold points and so must agree bit for bit."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_1909_01315_b200 as G
from paper_1909_01315_b200 import kernels
from oracle import gmp_oracle as O
from conftest import assert_close32, to_np

pytestmark = pytest.mark.gpu
DEV = "cuda"
ROOT = Path(__file__).resolve().parents[1]


def hub_graph(n=40000, hub_deg=30000, seed=7):
    """Rows of every class: hubs (> HEAVY_ROW_THRESHOLD in-edges, ragged
    counts), medium rows (33..2048) and light rows (<= 32, many of degree
    0..2)."""
    rng = np.random.default_rng(seed)
    src, dst = [], []
    for v, k in ((0, hub_deg), (1, hub_deg - 7), (2, 5000 + 13)):
        src.append(rng.choice(n, size=k, replace=False))
        dst.append(np.full(k, v))
    med = rng.integers(33, 400, size=200)
    for i, k in enumerate(med):
        src.append(rng.integers(0, n, size=k))
        dst.append(np.full(k, 10 + i))
    light = rng.integers(0, 3, size=n - 300)
    src.append(rng.integers(0, n, size=int(light.sum())))
    dst.append(np.repeat(np.arange(300, n), light))
    s = np.concatenate(src).astype(np.int64)
    d = np.concatenate(dst).astype(np.int64)
    perm = rng.permutation(s.size)  # edge ids not grouped by destination
    return s[perm], d[perm], n


def cancelling_features(n, d, seed):
    """+-1e4 offsets that cancel in every hub row plus unit noise: the exact
    sums are O(100) while their terms are 1e4."""
    rng = np.random.default_rng(seed)
    sign = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)[:, None]
    return (1e4 * sign + rng.standard_normal((n, d))).astype(np.float32)


@pytest.fixture
def small_budget(monkeypatch):
    """Below X's size for d > 75 but above one 256 B-row tile slice of the
    40000-row graph (10.2 MB): 64-column tiles, the pipelined kernel."""
    monkeypatch.setattr(kernels, "_L2_BUDGET", 12 << 20)


@pytest.mark.parametrize("d", [16, 32, 64, 128, 200])  # 4 / 8 / 16 lanes per edge
@pytest.mark.parametrize("rho", ["sum", "mean"])
def test_pipe_copy_matches_oracle(small_budget, d, rho):
    s, dd, n = hub_graph()
    g = G.from_arrays(s, dd, num_nodes=n, device=DEV)
    x = np.random.default_rng(d).standard_normal((n, d)).astype(np.float32)
    Z, _ = G.gspmm(g, kernels.copy("src"), rho, X=torch.as_tensor(x, device=DEV))
    want, _ = O.gspmm(s, dd, n, "copy_lhs", "src", None, rho, X=x.astype(np.float64))
    assert_close32(to_np(Z), want)


@pytest.mark.parametrize("d", [16, 32, 64])
def test_pipe_exact_under_cancellation(small_budget, d):
    s, dd, n = hub_graph()
    g = G.from_arrays(s, dd, num_nodes=n, device=DEV)
    x = cancelling_features(n, d, 3)
    Z, _ = G.gspmm(g, kernels.copy("src"), "sum", X=torch.as_tensor(x, device=DEV))
    want, _ = O.gspmm(s, dd, n, "copy_lhs", "src", None, "sum", X=x.astype(np.float64))
    assert_close32(to_np(Z), want)
    # the bar is meaningful here: a plain fp32 sum of the hub row misses it
    hub = np.flatnonzero(dd == 0)
    naive = np.zeros(d, dtype=np.float32)
    for u in s[hub]:
        naive += x[u]
    assert not np.allclose(naive, want[0], rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("rho", ["sum", "mean"])
def test_pipe_u_mul_e_matches_oracle(small_budget, rho):
    s, dd, n = hub_graph(seed=11)
    g = G.from_arrays(s, dd, num_nodes=n, device=DEV)
    rng = np.random.default_rng(5)
    x = cancelling_features(n, 130, 4)  # tiled: w laid out in adjacency order, the pipe path
    w = rng.standard_normal((s.size, 1)).astype(np.float32)
    Z, _ = G.gspmm(g, kernels.mul("src", "edge"), rho, X=torch.as_tensor(x, device=DEV),
                   W=torch.as_tensor(w, device=DEV))
    want, _ = O.gspmm(s, dd, n, "mul", "src", "edge", rho, X=x.astype(np.float64),
                      W=w.astype(np.float64))
    assert_close32(to_np(Z), want)


def test_pipe_deterministic(small_budget):
    s, dd, n = hub_graph()
    g = G.from_arrays(s, dd, num_nodes=n, device=DEV)
    x = torch.as_tensor(cancelling_features(n, 130, 9), device=DEV)
    a, _ = G.gspmm(g, kernels.copy("src"), "sum", X=x)
    b, _ = G.gspmm(g, kernels.copy("src"), "sum", X=x)
    assert torch.equal(a, b)


_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import paper_1909_01315_b200 as G
from paper_1909_01315_b200 import kernels
from test_gpu_pipe import hub_graph, cancelling_features
kernels._L2_BUDGET = 12 << 20
s, d, n = hub_graph()
g = G.from_arrays(s, d, num_nodes=n, device="cuda")
x = torch.as_tensor(cancelling_features(n, 64, 3), device="cuda")
z, _ = G.gspmm(g, kernels.copy("src"), "sum", X=x)
np.save(sys.argv[2], z.cpu().numpy())
"""


def test_pipe_equals_burst_kernel_on_heavy_and_medium_rows(tmp_path):
    outs = {}
    for tag, env in (("pipe", {}), ("burst", {"GMP_NO_PIPE": "1"})):
        f = tmp_path / (tag + ".npy")
        e = dict(os.environ, **env)
        subprocess.run([sys.executable, "-c", _CHILD, str(ROOT), str(f)], check=True, env=e,
                       timeout=600)
        outs[tag] = np.load(f)
    s, dd, n = hub_graph()
    deg = np.bincount(dd, minlength=n)
    rows = np.flatnonzero(deg > 32)  # heavy and medium rows: same order, same folds
    assert rows.size > 100
    assert np.array_equal(outs["pipe"][rows], outs["burst"][rows])
    want, _ = O.gspmm(s, dd, n, "copy_lhs", "src", None, "sum",
                      X=cancelling_features(n, 64, 3).astype(np.float64))
    assert_close32(outs["burst"], want)


@pytest.mark.parametrize("d", [16, 32, 64])
@pytest.mark.parametrize("rho", ["max", "min"])
def test_pipe_extrema_bit_exact(small_budget, d, rho):
    """max / min of copy_u through the pipelined ring: values and arg edges
    (smallest edge id among ties) equal the reference's bit for bit, with
    many exact ties (values drawn from 7 levels)."""
    s, dd, n = hub_graph(seed=13)
    g = G.from_arrays(s, dd, num_nodes=n, device=DEV)
    rng = np.random.default_rng(d)
    x = rng.integers(-3, 4, size=(n, d)).astype(np.float32) * np.float32(0.5)
    Z, aux = G.gspmm(g, kernels.copy("src"), rho, X=torch.as_tensor(x, device=DEV))
    want, warg = O.gspmm(s, dd, n, "copy_lhs", "src", None, rho, X=x.astype(np.float64))
    assert np.array_equal(to_np(Z), want.astype(np.float32))
    assert np.array_equal(to_np(aux.arg_edge), warg)
