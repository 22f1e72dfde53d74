"""Experiment: does Morton-sorting the queries make the projection coherent?"""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_11498_b200 import BSplineCurve, prepare_curve
from oracle import prep as P


def morton(q, bits=21):
    lo = q.min(0)
    span = np.maximum(q.max(0) - lo, 1e-300)
    u = np.clip(((q - lo) / span * ((1 << bits) - 1)).astype(np.uint64), 0, (1 << bits) - 1)

    def spread(x):
        x = x & np.uint64(0x1fffff)
        x = (x | x << np.uint64(32)) & np.uint64(0x1f00000000ffff)
        x = (x | x << np.uint64(16)) & np.uint64(0x1f0000ff0000ff)
        x = (x | x << np.uint64(8)) & np.uint64(0x100f00f00f00f00f)
        x = (x | x << np.uint64(4)) & np.uint64(0x10c30c30c30c30c3)
        x = (x | x << np.uint64(2)) & np.uint64(0x1249249249249249)
        return x
    return spread(u[:, 0]) | spread(u[:, 1]) << np.uint64(1) | spread(u[:, 2]) << np.uint64(2)


p, knots, ctrl = P.clamped_uniform_curve(np.random.default_rng(0), 7, 512, 3)
prep = prepare_curve(BSplineCurve(p, knots, ctrl), 1e-4)
tab = prep.table
from paper_2504_11498_b200 import _lib as L
qh = np.random.default_rng(1).uniform(0, 1, (1_000_000, 3))
for name, fl, screen, n in (("screen wave", 0, True, 1_000_000),
                            ("screen fused", L.MREP_FUSED, True, 1_000_000),
                            ("screen fused nosort", L.MREP_FUSED | L.MREP_NO_SORT, True, 1_000_000),
                            ("dense", 0, False, 100_000)):
    q = torch.from_numpy(np.ascontiguousarray(qh[:n])).cuda()
    tab.project(q, screen=screen, extra_flags=fl)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record()
        tab.project(q, screen=screen, extra_flags=fl)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name:22s} n={n} {best:8.3f} ms  {n / best / 1e3:8.2f} M pts/s", flush=True)
