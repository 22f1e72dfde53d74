"""Free HBM before / after the cfg3 workload's preparation and cell build."""
import sys

import torch

sys.path.insert(0, ".")
print("free/total GB at start", [x / 2**30 for x in torch.cuda.mem_get_info()], flush=True)
import bench  # noqa: E402
wl = bench.CurveSetWorkload("cfg3", 0, 1, 0)
torch.cuda.synchronize()
print("after cfg3 prep + cells", [x / 2**30 for x in torch.cuda.mem_get_info()],
      "index GB", wl.cells_bytes / 2**30, "torch reserved GB", torch.cuda.memory_reserved() / 2**30)
