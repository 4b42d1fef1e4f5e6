"""Host->device copy rates for the e2e pipeline's transfer shapes: one 1-D
copy vs the pitched 2-D copy of a 256 B-wide column tile (n rows of 2408 B
pitch), and the same for device->host."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_1909_01315_b200 import pipeline  # noqa: E402

n, d = 232965, 602
xh = torch.randn(n, d).pin_memory()
zh = torch.empty(n, d).pin_memory()
xd = torch.empty(n, d, device="cuda")
td = torch.empty(n, 64, device="cuda")
s = torch.cuda.Stream()


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / reps


ms = timeit(lambda: xd.copy_(xh, non_blocking=True) if False else
            pipeline._copy2d(xd.data_ptr(), d * 4, xh.data_ptr(), d * 4, d * 4, n, 1, s))
print("H2D 1-D (as 2-D full rows) %.2f ms  %.1f GB/s" % (ms, n * d * 4 / ms / 1e6))
ms = timeit(lambda: pipeline._copy2d(td.data_ptr(), 256, xh.data_ptr(), d * 4, 256, n, 1, s))
print("H2D 2-D 256 B x %d rows %.2f ms  %.1f GB/s" % (n, ms, n * 256 / ms / 1e6))
ms = timeit(lambda: pipeline._copy2d(zh.data_ptr(), d * 4, td.data_ptr(), 256, 256, n, 2, s))
print("D2H 2-D 256 B x %d rows %.2f ms  %.1f GB/s" % (n, ms, n * 256 / ms / 1e6))
ms = timeit(lambda: pipeline._copy2d(zh.data_ptr(), d * 4, xd.data_ptr(), d * 4, d * 4, n, 2, s))
print("D2H 1-D %.2f ms  %.1f GB/s" % (ms, n * d * 4 / ms / 1e6))
