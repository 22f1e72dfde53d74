"""Packet tree walk vs cell index for the cfg2 / cfg5 curve (device time)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2504_11498_b200 import _lib as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
grids = [int(x) for x in sys.argv[2:]] or [64]
wl = bench.SingleCurve(cfg, 0, 1, 1000000)


def timeit(q, flags):
    for _ in range(3):
        wl.tab.project(q, extra_flags=flags)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(10):
        wl.tab.project(q, extra_flags=flags)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 10


for m in (131072, 1000000):
    q = wl.q[:m].contiguous()
    print(cfg, m, "packet", round(timeit(q, L.MREP_PACKET), 3), "ms")
for g in grids:
    import time
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    wl.tab.build_cells(g)
    torch.cuda.synchronize()
    print("grid", g, "build", round((time.perf_counter() - t0) * 1e3, 1), "ms",
          wl.tab.cells.numel() * 4 / 1e6, "MB")
    for m in (131072, 1000000):
        q = wl.q[:m].contiguous()
        print(cfg, m, "cells", g, round(timeit(q, L.MREP_CELLS), 3), "ms")
