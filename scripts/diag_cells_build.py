"""Build the cell index of the cfg5 table (memcheck target)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 16
wl = bench.SingleCurve("cfg5", 0, 1, 1000)
wl.tab.build_cells(g)
torch.cuda.synchronize()
print("built", g, wl.tab.cells.numel())
