"""cfg5 (10^5 cubics): cell grid size vs build cost, index bytes and
projection time of 4e6 queries."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2504_11498_b200 import _lib as L  # noqa: E402

wl = bench.SingleCurve("cfg5", 0, 1, 4000000)
tab = wl.tab
tab.CELL_MAX_BYTES = 64 << 30
q = wl.q
for g in [int(x) for x in sys.argv[1:]] or (128, 192, 256):
    tab.cells = None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tab.build_cells(g)
    torch.cuda.synchronize()
    bms = (time.perf_counter() - t0) * 1e3
    for _ in range(2):
        tab.project(q, extra_flags=L.MREP_CELLS)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(5):
        tab.project(q, extra_flags=L.MREP_CELLS)
    b.record()
    torch.cuda.synchronize()
    print(f"grid {g}: build {bms:.0f} ms, {tab.cells.numel() * 4 / 1e9:.2f} GB, "
          f"{a.elapsed_time(b) / 5:.2f} ms per 4e6 queries", flush=True)
