"""Seeded synthetic inputs for BASELINE.json configs C1 (Cora-shaped GCN) and
C2 (Pubmed-shaped GAT), regenerated identically by the golden generator and
by the tests (uniform multigraph rng.integers(0, n, m) as in
the reference's conftest.py:25-31; fp32-representable features)."""

import numpy as np

SAMPLE_ROWS = np.arange(0, 19717, 97)


def c1_inputs(seed=0):
    rng = np.random.default_rng(seed)
    n, m = 2708, 10556
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    x = (rng.random((n, 1433)) < 0.0127).astype(np.float32)
    labels = rng.integers(0, 7, n)
    return src, dst, n, x, labels


def c2_inputs(seed=1):
    rng = np.random.default_rng(seed)
    n, m = 19717, 88651
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    x = rng.random((n, 500), dtype=np.float32)
    u = rng.standard_normal((n, 64)).astype(np.float32)
    return src, dst, n, x, u
