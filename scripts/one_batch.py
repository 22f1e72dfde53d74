"""One cfg3 batched projection (10^4 curves, 10^6 queries) for ncu captures
(after one warm-up call; the measured call is the NVTX range "timed")."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

wl = bench.CurveSetWorkload("cfg3", 0, 1, 0)
wl.step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("timed")
wl.step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
