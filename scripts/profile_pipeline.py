"""One projection call (after warm-up) for ncu launch lists: --fused or wavefront."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_11498_b200 import BSplineCurve, prepare_curve
from paper_2504_11498_b200 import _lib as L
from oracle import prep as P
fl = L.MREP_FUSED if "--fused" in sys.argv else 0
p, knots, ctrl = P.clamped_uniform_curve(np.random.default_rng(0), 7, 512, 3)
prep = prepare_curve(BSplineCurve(p, knots, ctrl), 1e-4)
q = torch.from_numpy(np.random.default_rng(1).uniform(0, 1, (1_000_000, 3))).cuda()
for _ in range(3):
    prep.table.project(q, extra_flags=fl)
torch.cuda.synchronize()
