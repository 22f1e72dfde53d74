"""Breakdown of prepare_curve_set for the cfg3 set (host vs device stages)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_11498_b200 import _lib as L  # noqa: E402
from paper_2504_11498_b200.batch import prepare_curve_set  # noqa: E402
from paper_2504_11498_b200.core import validate_curve  # noqa: E402
from paper_2504_11498_b200.decompose import DeviceCurves, decompose_device  # noqa: E402
from paper_2504_11498_b200.fixtures import mixed_curve_batch  # noqa: E402
from paper_2504_11498_b200.reduce_approx import approximate_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
t0 = time.perf_counter()
curves = mixed_curve_batch(n)
t1 = time.perf_counter()
print(f"generate {n} curves: {(t1 - t0) * 1e3:.0f} ms")
prepare_curve_set(curves[:50])  # warm
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    for c in curves:
        validate_curve(c)
    t1 = time.perf_counter()
    dc = DeviceCurves(curves)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    dec = decompose_device(dc)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    res = approximate_device(dec["rows"], dec["row_ofs"], dec["iv"], dec["curve"], dec["nseg"], 3,
                             1e-4, 4096 * n)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    out = res.fetch()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    cs = prepare_curve_set(curves)
    torch.cuda.synchronize()
    t6 = time.perf_counter()
    print(f"validate {1e3 * (t1 - t0):.0f} ms | DeviceCurves {1e3 * (t2 - t1):.0f} | decompose "
          f"{1e3 * (t3 - t2):.0f} | approximate {1e3 * (t4 - t3):.0f} | fetch {1e3 * (t5 - t4):.0f}"
          f" | full prepare_curve_set {1e3 * (t6 - t5):.0f} ms ({cs.num_segments} cubics)")
