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


def c2_weights(init_gat):
    """C2 head weights: the reference's init_gat(rng 7, 500, 8, 8), rounded to
    fp32 so the fp32 and fp64 runs and the reference all see the same
    (exactly representable) values - the fp32 parity protocol."""
    params = init_gat(np.random.default_rng(7), 500, 8, 8)
    for hp in params.heads:
        hp.W, hp.a_l, hp.a_r = (np.asarray(a, np.float32).astype(np.float64)
                                for a in (hp.W, hp.a_l, hp.a_r))
    return params
