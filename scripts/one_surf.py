"""One cfg4 / cfg4q surface projection (for ncu captures)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 0
wl = bench.SurfaceWorkload(cfg, 0, 1, 1000000)
for _ in range(warm):
    wl.step()
torch.cuda.synchronize()
wl.step()
torch.cuda.synchronize()
