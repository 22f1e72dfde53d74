"""Traversal-variant A/B correctness (MREP_TRAV_DMMA, MREP_SET_SCAN, ...): project the bench inputs of a config with
the given environment and save (t, foot, dist, seg); compare two saves.
    python scripts/dmma_check.py cfg2 out.npz [n]      |  python scripts/dmma_check.py cmp a.npz b.npz"""
import sys

import numpy as np

if sys.argv[1] == "cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in ("t", "foot", "dist", "seg"):
        same = np.array_equal(a[k], b[k], equal_nan=True)
        print(k, "bit-identical" if same else f"DIFFERENT ({int(np.sum(a[k] != b[k]))})")
    print("cand mean", a["cand"].mean(), b["cand"].mean())
    sys.exit(0)
import torch  # noqa: E402
sys.path.insert(0, ".")
import bench  # noqa: E402

cfg = sys.argv[1]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 0
wl = (bench.NearestWorkload if cfg == "cfg6" else bench.CurveSetWorkload if cfg == "cfg3"
      else bench.SingleCurve)(cfg, 0, 1, n)
out = wl.step()
t, foot, dist, cand, seg = (x.cpu().numpy() for x in out[:5])
np.savez(sys.argv[2], t=t, foot=foot, dist=dist, cand=cand, seg=seg)
print("saved", sys.argv[2], len(t))
