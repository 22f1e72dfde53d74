"""Minimal driver for ncu captures of the projection kernels.

    python scripts/profile_kernels.py --mode screen|dense [--n N]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2504_11498_b200 import _device as D  # noqa: E402
from paper_2504_11498_b200 import BSplineCurve, prepare_curve  # noqa: E402
from oracle import prep as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="screen")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--reps", type=int, default=4)
a = ap.parse_args()
p, knots, ctrl = P.clamped_uniform_curve(np.random.default_rng(0), 7, 512, 3)
prep = prepare_curve(BSplineCurve(p, knots, ctrl), 1e-4)
n = a.n or (1_000_000 if a.mode == "screen" else 100_000)
q = torch.from_numpy(np.random.default_rng(1).uniform(0, 1, (n, 3))).cuda()
for _ in range(a.reps):
    prep.table.project(q, screen=(a.mode == "screen"))
torch.cuda.synchronize()
print("done", a.mode, n)
