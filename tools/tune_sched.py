"""Schedule-threshold sweep (heavy / light row thresholds of gmp_build_schedule):
python tools/tune_sched.py HEAVY LIGHT  -> times copy_u+sum d=602 / d=16 and a GAT epoch."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01315_b200 as G  # noqa: E402
from paper_1909_01315_b200 import graph as GR, kernels, layers  # noqa: E402

GR.HEAVY_ROW_THRESHOLD, GR.LIGHT_ROW_THRESHOLD = int(sys.argv[1]), int(sys.argv[2])
kernels.HEAVY_ROW_THRESHOLD, kernels.LIGHT_ROW_THRESHOLD = GR.HEAVY_ROW_THRESHOLD, GR.LIGHT_ROW_THRESHOLD
dev = torch.device("cuda")
s, d = G.generators.power_law_edges(232965, 492, seed=0)
g = G.from_arrays(s, d, num_nodes=232965, device=dev)
gen = torch.Generator(device=dev).manual_seed(0)
X = torch.randn((232965, 602), generator=gen, device=dev)
X16 = torch.randn((232965, 16), generator=gen, device=dev)
labels = torch.randint(0, 41, (232965,), generator=gen, device=dev)
gat = layers.GATModel([602, 16, 16, 41], heads=1, seed=0, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


print("heavy=%s light=%s  copy602 %.3f  copy16 %.3f  gat %.3f" % (
    sys.argv[1], sys.argv[2], t(lambda: G.gspmm(g, kernels.copy("src"), "sum", X=X)),
    t(lambda: G.gspmm(g, kernels.copy("src"), "sum", X=X16)),
    t(lambda: layers.train_epoch(g, X, labels, gat, 0.01))))
