"""Device time per call of small batches (cfg1 curve): wavefront vs the fused
single-kernel screened path (MREP_FUSED), CUDA events, median of 50."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2504_11498_b200 import _lib as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
wl = bench.SingleCurve(cfg, 0, 1, 0)
sizes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1000, 4000, 10000, 30000]
for n in sizes:
    q = wl.q[:n].contiguous() if n <= wl.q.shape[0] else wl.q.repeat((n + wl.q.shape[0] - 1) // wl.q.shape[0], 1)[:n].contiguous()
    for name, fl in (("wave", 0), ("fused", L.MREP_FUSED)) if n <= 100000 else (("wave", 0),):
        flags = wl.tab._cell_flag(n, True) | fl
        for _ in range(5):
            wl.tab.project(q, extra_flags=flags)
        ts = []
        for _ in range(50):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            wl.tab.project(q, extra_flags=flags)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        print(f"{cfg} n={n} {name}: {ts[len(ts) // 2]:.4f} ms", flush=True)
