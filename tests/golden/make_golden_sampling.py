"""Golden outputs of the reference's neighbor_sample (graph.py:231-286) for
the cases where the draw is not random (fanout >= every seed's in-degree):
then the reference's result is fully determined by its relabelling rules
(seeds first in first-occurrence order, new nodes ascending, picks ascending
per seed) and the device sampler must reproduce it exactly.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden_sampling.py   -> tests/golden/sampling.npz
"""

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")


def cases():
    """(src, dst, n, seeds) inputs, regenerated from seeds on both sides."""
    out = []
    rng = np.random.default_rng(2024)
    for i in range(6):
        n = int(rng.integers(5, 60))
        m = int(rng.integers(0, 400))
        s = rng.integers(0, n, m)
        d = rng.integers(0, n, m)
        seeds = rng.integers(0, n, int(rng.integers(1, 12)))
        out.append((s, d, n, seeds))
    return out


def main():
    import graphmp as G
    res = {}
    for i, (s, d, n, seeds) in enumerate(cases()):
        g = G.from_arrays(s.astype(np.uint32), d.astype(np.uint32), num_nodes=n)
        sub = G.neighbor_sample(g, seeds.tolist(), fanout=10_000, rng_seed=i)
        su, de, _ = sub.graph.coo()
        res["s%d/node_ids" % i] = sub.parent_node_ids.astype(np.int64)
        res["s%d/edge_ids" % i] = sub.parent_edge_ids.astype(np.int64)
        res["s%d/sub_src" % i] = su.astype(np.int64)
        res["s%d/sub_dst" % i] = de.astype(np.int64)
    np.savez_compressed(HERE / "sampling.npz", **res)
    print("wrote", HERE / "sampling.npz", len(res), "arrays")


if __name__ == "__main__":
    main()
