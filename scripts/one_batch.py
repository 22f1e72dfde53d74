"""One cfg3 batched projection (10^4 curves, 10^6 queries) for ncu captures."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

wl = bench.CurveSetWorkload("cfg3", 0, 1, 0)
torch.cuda.synchronize()
wl.step()
torch.cuda.synchronize()
