"""Per-stage device times (MREP_TIMING) of the cfg2 projection vs batch size."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2504_11498_b200 import _lib as L  # noqa: E402

wl = bench.SingleCurve(sys.argv[1] if len(sys.argv) > 1 else "cfg2", 0, 1, 0)
flags = wl.tab._cell_flag(1 << 20, True)
print("stages: sort traverse pairs clip select fallback")
for m in (65536, 125000, 250000, 500000, 1000000):
    q = wl.q[:m].contiguous()
    acc = np.zeros(6)
    for r in range(8):
        wl.tab.project(q, extra_flags=flags | L.MREP_TIMING)
        buf = (ctypes.c_double * 8)()
        L.lib().mrep_last_stage_times(buf, 8)
        if r >= 3:
            acc += np.array(buf[:6]) / 5
    print(m, np.round(acc, 4), round(acc.sum(), 4))
