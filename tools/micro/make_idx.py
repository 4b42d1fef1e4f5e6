"""Index streams for l2gather_file: the CSC-ordered sources of the
Reddit-shaped graph (what the row kernel gathers), the same multiset
shuffled, and uniform random rows."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_1909_01315_b200 import generators  # noqa: E402

cache = Path("/tmp/pl_edges.npz")
if cache.exists():
    z = np.load(cache)
    s, d = z["s"], z["d"]
else:
    s, d = generators.power_law_edges(232965, 492, seed=0)
    np.savez(cache, s=s, d=d)
order = np.lexsort((s, d))
csc = s[order].astype(np.uint32)
csc.tofile("/tmp/idx_csc.bin")
rng = np.random.default_rng(0)
rng.permutation(csc).tofile("/tmp/idx_shuf.bin")
rng.integers(0, 232965, size=csc.size, dtype=np.uint32).tofile("/tmp/idx_unif.bin")
