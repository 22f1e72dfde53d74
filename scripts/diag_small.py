"""Device time of small batches (cfg1 curve): wavefront vs fused kernel, sort on/off."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2504_11498_b200 import _lib as L  # noqa: E402

wl = bench.SingleCurve(sys.argv[1] if len(sys.argv) > 1 else "cfg1", 0, 1, 0)
for n in (2000, 10000, 16384, 32768):
    q = wl.q[:n].contiguous() if n <= len(wl.q) else wl.q.repeat(n // len(wl.q) + 1, 1)[:n].contiguous()
    for name, fl in (("wave", 0), ("wave-nosort", L.MREP_NO_SORT), ("fused", L.MREP_FUSED),
                     ("fused-nosort", L.MREP_FUSED | L.MREP_NO_SORT)):
        for _ in range(5):
            wl.tab.project(q, extra_flags=fl)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(50):
            wl.tab.project(q, extra_flags=fl)
        b.record()
        torch.cuda.synchronize()
        print(n, name, round(a.elapsed_time(b) / 50, 4), "ms")
