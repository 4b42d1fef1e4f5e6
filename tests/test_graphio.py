"""graphio: files written by the reference (tests/golden/io, made by
tests/golden/make_golden_io.py) load bit-exactly, and this package's writers
reproduce them byte for byte (graphio.py:58-113 formats). CPU tensors here;
the -m gpu variant loads onto cuda and runs a kernel on the loaded graph."""

from pathlib import Path

import numpy as np
import pytest
import torch

import paper_1909_01315_b200 as G
from paper_1909_01315_b200 import graphio
from conftest import to_np

IO = Path(__file__).resolve().parent / "golden" / "io"


def expect():
    e = np.load(IO / "expect.npz")
    return e["src"], e["dst"], int(e["n"]), e["x"]


def test_read_reference_files():
    s, d, n, x = expect()
    g = graphio.read_graph_binary(IO / "g.grf1", device="cpu")
    assert g.num_nodes == n and np.array_equal(to_np(g.src), s) and np.array_equal(to_np(g.dst), d)
    g2 = graphio.read_edge_list(IO / "g.tsv", device="cpu")
    assert g2.num_nodes == n and np.array_equal(to_np(g2.src), s)
    xf = graphio.read_features_binary(IO / "x.fmx1", device="cpu", dtype=torch.float64)
    assert np.array_equal(to_np(xf), x)
    xc = graphio.read_features_csv(IO / "x.csv", device="cpu", dtype=torch.float64)
    assert np.array_equal(to_np(xc), x)
    assert graphio.read_loss_curve(IO / "loss.csv") == [1.5, 1.25, 0.875]


def test_writers_byte_identical(tmp_path):
    s, d, n, x = expect()
    g = G.Graph(s.astype(np.int64), d.astype(np.int64), n, device="cpu")
    for name, write, arg in (("g.grf1", graphio.write_graph_binary, g),
                             ("g.tsv", graphio.write_edge_list, g),
                             ("x.fmx1", graphio.write_features_binary, x),
                             ("x.csv", graphio.write_features_csv, x),
                             ("loss.csv", graphio.write_loss_curve, [1.5, 1.25, 0.875])):
        write(tmp_path / name, arg)
        assert (tmp_path / name).read_bytes() == (IO / name).read_bytes(), name


def test_errors(tmp_path):
    bad = tmp_path / "bad.grf1"
    bad.write_bytes(b"XXXX" + bytes(16))
    with pytest.raises(ValueError, match="bad magic"):
        graphio.read_graph_binary(bad, device="cpu")
    trunc = tmp_path / "t.grf1"
    trunc.write_bytes((IO / "g.grf1").read_bytes()[:-8])
    with pytest.raises(ValueError, match="truncated"):
        graphio.read_graph_binary(trunc, device="cpu")
    tf = tmp_path / "t.fmx1"
    tf.write_bytes((IO / "x.fmx1").read_bytes()[:-8])
    with pytest.raises(ValueError, match="truncated"):
        graphio.read_features_binary(tf, device="cpu")
    el = tmp_path / "e.tsv"
    el.write_text("0\t1\n2 3 4\n")
    with pytest.raises(ValueError, match="expected"):
        graphio.read_edge_list(el, device="cpu")
    empty = tmp_path / "empty.grf1"
    graphio.write_graph_binary(empty, G.Graph(np.zeros(0, np.int64), np.zeros(0, np.int64), 4,
                                              device="cpu"))
    assert graphio.read_graph_binary(empty, device="cpu").num_edges == 0


@pytest.mark.gpu
def test_load_to_device_and_aggregate():
    from paper_1909_01315_b200 import kernels
    from oracle import gmp_oracle as O
    s, d, n, x = expect()
    g = graphio.read_graph_binary(IO / "g.grf1", device="cuda")
    xf = graphio.read_features_binary(IO / "x.fmx1", device="cuda")
    assert g.src.is_cuda and xf.is_cuda and xf.dtype == torch.float32
    z, _ = G.gspmm(g, kernels.copy("src"), "sum", X=xf)
    want, _ = O.gspmm(s, d, n, "copy_lhs", "src", None, "sum", X=x.astype(np.float32))
    assert np.allclose(to_np(z), want, rtol=1e-5, atol=1e-6)
