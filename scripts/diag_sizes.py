"""Device time of one screened projection vs batch size (cfg2 curve)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

wl = bench.SingleCurve("cfg2", 0, 1, 0)
for m in [int(x) for x in sys.argv[1:]] or (65536, 131072, 262144, 458752, 1000000):
    q = wl.q[:m].contiguous()
    for _ in range(3):
        wl.tab.project(q)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(20):
        wl.tab.project(q)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    print(f"n={m}: {ms:.3f} ms  {m / ms / 1e3:.1f} M pts/s")
