"""Dump cfg4 / cfg4q surface projections (u, v, foot, dist, patch) to an npz
(A/B bitwise comparisons of two library builds via MREP_LIB)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402

out = sys.argv[1]
res = {}
for cfg in ("cfg4", "cfg4q"):
    wl = bench.SurfaceWorkload(cfg, 0, 1, 300000)
    for i, a in enumerate(wl.step()):
        res[f"{cfg}_{i}"] = a.cpu().numpy()
np.savez(out, **res)
