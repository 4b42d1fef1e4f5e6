import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1909_01315_b200 as G
from paper_1909_01315_b200 import layers
z = np.load('/tmp/pl_edges.npz'); s, d = z['s'], z['d']
n = 232965
dev = torch.device('cuda')
g = G.from_arrays(s, d, num_nodes=n, device=dev)
gen = torch.Generator(device=dev); gen.manual_seed(0)
X = torch.randn((n, 602), generator=gen, device=dev)
labels = torch.randint(0, 41, (n,), generator=gen, device=dev)
for name, model in (("gat", layers.GATModel([602, 16, 16, 41], heads=1, seed=0, device=dev)),
                    ("gcn", layers.GCNModel([602, 16, 41], seed=0, device=dev))):
    for _ in range(3): layers.train_epoch(g, X, labels, model, 0.01)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as p:
        for _ in range(3): layers.train_epoch(g, X, labels, model, 0.01)
        torch.cuda.synchronize()
    print("==", name)
    print(p.key_averages().table(sort_by="cuda_time_total", row_limit=14, max_name_column_width=70))
