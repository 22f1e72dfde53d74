"""One screened cfg2 projection of n queries (for launch-list profiling)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
wl = bench.SingleCurve("cfg2", 0, 1, 0)
q = wl.q[:n].contiguous()
for _ in range(3):
    wl.tab.project(q)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("measured")
wl.tab.project(q)
torch.cuda.synchronize()
