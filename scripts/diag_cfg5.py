import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_11498_b200 import BSplineCurve, prepare_curve, _lib as L
from paper_2504_11498_b200.fixtures import random_clamped_curve
c = random_clamped_curve(np.random.default_rng(0), 3, 100_003, 3, uniform_knots=True)
prep = prepare_curve(c, 1e-4)
print("S", prep.num_segments, "seg len median", np.median(np.linalg.norm(prep.seg_pts[:, 3] - prep.seg_pts[:, 0], axis=1)))
q = torch.from_numpy(np.random.default_rng(1).uniform(0, 1, (1_000_000, 3))).cuda()
cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
out = prep.table.project(q, counters=cnt)
torch.cuda.synchronize()
c7 = int(cnt[7].item())
print("counters", cnt.cpu().numpy().tolist(), "emitted pairs/surv/cand (x1024):", c7 & 0x1fffff, (c7 >> 21) & 0x1fffff, (c7 >> 42) & 0x1fffff)
seg = out[4].cpu().numpy(); d = out[2].cpu().numpy()
print("dist median", np.median(d), "max", d.max(), "neg seg", (seg < 0).sum())
