"""Timeline of the e2e host pipeline (pipeline.gspmm_host's schedule,
replicated with events): when each tile's H2D, kernel and D2H start / end."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1909_01315_b200 as G  # noqa: E402
from paper_1909_01315_b200 import kernels, pipeline  # noqa: E402

z = np.load("/tmp/pl_edges.npz")
n, d = 232965, 602
g = G.from_arrays(z["s"], z["d"], num_nodes=n, device="cuda")
g.to_csc().schedule()
xh = torch.randn(n, d).pin_memory()
zh = torch.empty(n, d).pin_memory()
p = pipeline.HostPipeline("cuda", persist_l2=False)
tiles, tw = pipeline.tile_bounds(d, 4)
Xd = p.buffer("X", (len(tiles), n, tw), torch.float32, zero=True)
Zd = p.buffer("Z", (len(tiles), n, tw), torch.float32)
comp = torch.cuda.current_stream()
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
for rep in range(3):
    t0 = E(); t0.record(comp)
    p.h2d.wait_stream(comp)
    hs, he, ks, ke, ds, de = [], [], [], [], [], []
    for t, (c0, c1) in enumerate(tiles):
        a, b = E(), E()
        a.record(p.h2d)
        pipeline._copy2d(Xd[t].data_ptr(), tw * 4, xh.data_ptr() + c0 * 4, d * 4, (c1 - c0) * 4, n, 1, p.h2d)
        b.record(p.h2d)
        hs.append(a); he.append(b)
    for t, (c0, c1) in enumerate(tiles):
        comp.wait_event(he[t])
        w = -(-(c1 - c0) // 4) * 4
        a, b = E(), E()
        a.record(comp)
        kernels._gspmm_launch(g, kernels.copy("src"), "sum", Xd[t][:, :w], None, None, w, out=Zd[t][:, :w])
        b.record(comp)
        ks.append(a); ke.append(b)
    for t, (c0, c1) in enumerate(tiles):
        p.d2h.wait_event(ke[t])
        a, b = E(), E()
        a.record(p.d2h)
        pipeline._copy2d(zh.data_ptr() + c0 * 4, d * 4, Zd[t].data_ptr(), tw * 4, (c1 - c0) * 4, n, 2, p.d2h)
        b.record(p.d2h)
        ds.append(a); de.append(b)
    comp.wait_stream(p.d2h)
    te = E(); te.record(comp)
    te.synchronize()
    if rep < 2:
        continue
    f = lambda e: t0.elapsed_time(e)  # noqa: E731
    for t in range(len(tiles)):
        print("tile %d  H2D %6.2f-%6.2f  kernel %6.2f-%6.2f  D2H %6.2f-%6.2f" % (
            t, f(hs[t]), f(he[t]), f(ks[t]), f(ke[t]), f(ds[t]), f(de[t])))
    print("total %.2f ms" % f(te))
