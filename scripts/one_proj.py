"""One screened cfg2 projection of n queries (for ncu launch lists).
EXTRA_FLAGS=<int> adds mrep flags (e.g. 512 = MREP_CAND_EXACT)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 125000
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl = bench.SingleCurve("cfg2", 0, 1, 0)
flags = wl.tab._cell_flag(1 << 20, True) | int(os.environ.get("EXTRA_FLAGS", "0"))
if flags & 1024:  # MREP_CAND_CELLS: build the table's cand cell index first
    wl.tab.build_cand_cells()
q = wl.q[:n].contiguous()
for _ in range(warm):
    wl.tab.project(q, extra_flags=flags)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("timed")
wl.tab.project(q, extra_flags=flags)
torch.cuda.synchronize()
