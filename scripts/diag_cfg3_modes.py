"""cfg3 (10^4 curves, 10^6 queries): device time per traversal mode."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2504_11498_b200 import _lib as L  # noqa: E402

wl = bench.CurveSetWorkload("cfg3", 0, 1, 0)
for name, f in (("auto", 0), ("group", L.MREP_GROUP), ("lane", L.MREP_PER_LANE),
                ("packet", L.MREP_PACKET)):
    for _ in range(3):
        wl.step(extra_flags=f)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(10):
        wl.step(extra_flags=f)
    b.record()
    torch.cuda.synchronize()
    print(name, round(a.elapsed_time(b) / 10, 3), "ms", flush=True)
