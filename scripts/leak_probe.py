import sys, gc
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2504_11498_b200 import prepare_curve
from paper_2504_11498_b200 import reduce_approx as R
from paper_2504_11498_b200.fixtures import random_clamped_curve
orig = R.ApproxResult.__del__
def dbg(self):
    print("ApproxResult.__del__", self.handle, file=sys.stderr)
    orig(self)
R.ApproxResult.__del__ = dbg
prepare_curve(random_clamped_curve(np.random.default_rng(0), 5, 40, 3, uniform_knots=True))
gc.collect()
torch.cuda.synchronize()
print("done", file=sys.stderr)
objs = [o for o in gc.get_objects() if isinstance(o, R.ApproxResult)]
print("live ApproxResult:", len(objs), file=sys.stderr)
for o in objs[:3]:
    for r in gc.get_referrers(o):
        print("  referrer:", type(r), (list(r.keys())[:20] if isinstance(r, dict) else str(r)[:200]), file=sys.stderr)
