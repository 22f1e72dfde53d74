"""One preparation call (cfg2: prepare_curve of the degree-7 curve; cfg3:
prepare_curve_set of the 10^4 mixed curves) inside the NVTX range "timed",
after a warm-up call, for ncu launch lists / captures."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2504_11498_b200 import BSplineCurve, prepare_curve, prepare_curve_set  # noqa: E402
from paper_2504_11498_b200.fixtures import mixed_curve_batch  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
if cfg == "cfg3":
    curves = mixed_curve_batch(bench.CONFIGS["cfg3"]["curves"])
    run = lambda: prepare_curve_set(curves, 1e-4).free()  # noqa: E731
else:
    cv = BSplineCurve(*bench.make_curve(cfg))
    run = lambda: prepare_curve(cv, 1e-4)  # noqa: E731
run()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("timed")
run()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
