"""Timeline of the pipelined host-buffer call (MREP_E2E_TRACE=1 prints per
chunk upload / kernels / download end times): python scripts/e2e_trace.py [cfg] [reps]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
os.environ.setdefault("MREP_E2E_TRACE", "1")
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl = bench.SingleCurve(cfg, 0, 1, 0)
wl.pinned()
n = wl.q.shape[0]
outs = (torch.empty(n, dtype=torch.float64).pin_memory(),
        torch.empty((n, 3), dtype=torch.float64).pin_memory(),
        torch.empty(n, dtype=torch.float64).pin_memory(),
        torch.empty(n, dtype=torch.int64).pin_memory(),
        torch.empty(n, dtype=torch.int32).pin_memory())
onp = tuple(o.numpy() for o in outs)
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    wl.host(onp)
    print(f"rep {r}: {1e3 * (time.perf_counter() - t0):.3f} ms wall", file=sys.stderr, flush=True)
