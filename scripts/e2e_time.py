"""Mean wall time of the host-buffer call (as bench.py's e2e leg): python scripts/e2e_time.py cfg reps"""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
wl = (bench.CurveSetWorkload if cfg == "cfg3" else bench.SingleCurve)(cfg, 0, 1, 0)
wl.pinned()
n = wl.n
outs = (torch.empty(n, dtype=torch.float64).pin_memory(),
        torch.empty((n, 3), dtype=torch.float64).pin_memory(),
        torch.empty(n, dtype=torch.float64).pin_memory(),
        torch.empty(n, dtype=torch.int64).pin_memory(),
        torch.empty(n, dtype=torch.int32).pin_memory())
onp = tuple(o.numpy() for o in outs)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for _ in range(3):
    wl.host(onp)
ts = []
for _ in range(reps):
    flush.fill_(1.0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    wl.host(onp)
    ts.append(time.perf_counter() - t0)
print(f"mean {1e3 * statistics.mean(ts):.3f} ms  median {1e3 * statistics.median(ts):.3f} ms  "
      f"min {1e3 * min(ts):.3f} ms  ({n / statistics.mean(ts):.3e} pts/s)")
