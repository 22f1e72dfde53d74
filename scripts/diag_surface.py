"""Surface pipeline work counters + stage times (cfg4 / cfg4q), tree walk vs
cell index at several grid sizes."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2504_11498_b200 import _lib as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
grids = [int(x) for x in sys.argv[2:]] or [64]
wl = bench.SurfaceWorkload(cfg, 0, 1, 1000000)
tab = wl.tab


def run(flags):
    cnt = torch.zeros(L.NUM_COUNTERS, dtype=torch.int64, device="cuda")
    tab.project(wl.q, counters=cnt, extra_flags=flags)
    for _ in range(3):
        tab.project(wl.q, extra_flags=flags)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(10):
        tab.project(wl.q, extra_flags=flags)
    b.record()
    torch.cuda.synchronize()
    tab.project(wl.q, extra_flags=flags | L.MREP_TIMING)
    buf = (ctypes.c_double * 8)()
    L.lib().mrep_last_stage_times(buf, 8)
    c = cnt.cpu().numpy() / len(wl.q)
    return a.elapsed_time(b) / 10, np.round(buf[:6], 3), dict(
        pairs=c[L.CNT_PAIRS], iters=c[L.CNT_CLIP_ITERS], seeds=c[L.CNT_SEAMS],
        boxes=c[L.CNT_BOXES])


tab.use_cells = False
print(cfg, "tree", run(0))
tab.use_cells = True
for g in grids:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tab.build_cells(g)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    print(cfg, "grid", g, "build", round(ms, 1), "ms", tab.cells.numel() * 4 / 1e6, "MB",
          run(L.MREP_CELLS))
