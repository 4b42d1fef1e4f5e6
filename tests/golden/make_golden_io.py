"""GRF1 / FMX1 / edge-list / CSV files written by the reference's graphio
(/root/reference/pkg/src/graphmp/graphio.py), so tests/test_graphio.py can
check that this package reads the reference's files and writes byte-identical
ones without /root/reference at test time.

Run in the build container:  python tests/golden/make_golden_io.py
"""

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent / "io"
sys.path.insert(0, "/root/reference/pkg/src")


def main():
    from graphmp import graphio, graph
    HERE.mkdir(exist_ok=True)
    rng = np.random.default_rng(11)
    n, m = 37, 211
    s = rng.integers(0, n, m).astype(np.uint32)
    d = rng.integers(0, n, m).astype(np.uint32)
    g = graph.Graph(s, d, n)
    graphio.write_graph_binary(HERE / "g.grf1", g)
    graphio.write_edge_list(HERE / "g.tsv", g)
    x = rng.standard_normal((n, 5))
    graphio.write_features_binary(HERE / "x.fmx1", x)
    graphio.write_features_csv(HERE / "x.csv", x)
    graphio.write_loss_curve(HERE / "loss.csv", [1.5, 1.25, 0.875])
    np.savez(HERE / "expect.npz", src=s, dst=d, n=n, x=x)


if __name__ == "__main__":
    main()
