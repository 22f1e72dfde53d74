"""Parity at the bench's own scale: the exact inputs bench.py times.

* cfg5 (BASELINE configs[4]): random_clamped_curve(default_rng(0), 3, 100003)
  -> 10^5 cubics, the default cell index (384^3 from 2^16 cubics), the rank-0 shard of 10^8
  uniform queries (default_rng(1)), all projected on the GPU;
* cfg3 (BASELINE configs[2]): mixed_curve_batch(10_000) prepared as one
  device set (3.96 M cubics), 10^6 queries, 100 per curve, one batched call.

A stratified subsample of each run (random queries + seam winners + the
farthest queries + the ones whose screened walk examined the most) is checked
against the pinned C oracle (brute force over every cubic of the query's
curve): t within 1e-6, distance within 1e-9 relative, winning segment EXACT
except where the oracle itself finds another segment within dmin + 2e-12, and
the knot span of t* (core.py:108-112) exact.
"""
import os
import sys

import numpy as np
import pytest

from conftest import ROOT, assert_parity

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _strata(rng, n, t, dist, cand, seam_t, k):
    """Indices: k random, k seam winners, k farthest, k most-examined."""
    pick = [rng.choice(n, k, replace=False)]
    seam_win = np.nonzero(np.isin(t, seam_t))[0]
    if seam_win.size:
        pick.append(rng.choice(seam_win, min(k, seam_win.size), replace=False))
    pick.append(np.argpartition(dist, n - k)[n - k:])
    pick.append(np.argpartition(cand, n - k)[n - k:])
    return np.unique(np.concatenate(pick))


def test_cfg5_bench_inputs_vs_oracle(gpu, oracle_lib):
    import torch
    import bench
    from paper_2504_11498_b200 import BSplineCurve, prepare_curve
    p, knots, ctrl = bench.make_curve("cfg5")
    prep = prepare_curve(BSplineCurve(p, knots, ctrl), 1e-4)
    assert prep.num_segments == 100_000
    tab = prep.table
    tab._cell_flag(1 << 27, True)  # what bench.py does: the default index
    assert tab.cells is not None
    n = bench.CONFIGS["cfg5"]["n"]
    q_host = bench.make_queries("cfg5", 0, n)
    q = torch.from_numpy(q_host).cuda()
    t, foot, dist, cand, seg, _, _ = tab.project(q)
    t, dist, cand, seg = (x.cpu().numpy() for x in (t, dist, cand, seg))
    del q
    torch.cuda.empty_cache()
    idx = _strata(np.random.default_rng(5), n, t, dist, cand, prep.seam_t, 500)
    o = oracle_lib.project_block(prep.seg_pts, prep.seg_ta, prep.seg_tb, prep.seam_t,
                                 prep.seam_pt, q_host[idx], workers=os.cpu_count() or 1)
    span = prep.knot_spans(t[idx])
    ties = assert_parity(t[idx], dist[idx], seg[idx], o, span=span, knots=knots, degree=p)
    assert ties <= len(idx) // 100
    # the screened walk examined a tiny fraction of what brute force does
    assert float(cand.mean()) < 100


def test_cfg3_bench_inputs_vs_oracle(gpu, oracle_lib):
    import bench
    from paper_2504_11498_b200 import prepare_curve_set
    from paper_2504_11498_b200.fixtures import mixed_curve_batch
    cfg = bench.CONFIGS["cfg3"]
    curves = mixed_curve_batch(cfg["curves"])
    cset = prepare_curve_set(curves, 1e-4)
    n = cfg["n"]
    rng = np.random.default_rng(1)  # bench.CurveSetWorkload, rank 0
    cid = (np.arange(n) % cfg["curves"]).astype(np.int32)
    rng.shuffle(cid)
    q = rng.uniform(0.0, 1.0, (n, 3))
    t, foot, dist, cand, seg = (x.cpu().numpy() for x in cset.project_device(q, cid))
    spans = cset.knot_spans(t, cid)
    counts = cset.segment_counts()
    chosen = set(range(0, len(curves), 25)) | set(np.argsort(counts)[-20:].tolist())
    workers = os.cpu_count() or 1
    ties = checked = 0
    for c in sorted(chosen):
        m = np.nonzero(cid == c)[0]
        pc = cset[c]
        o = oracle_lib.project_block(pc.seg_pts, pc.seg_ta, pc.seg_tb, pc.seam_t, pc.seam_pt,
                                     q[m], workers=workers)
        cv = curves[c]
        ties += assert_parity(t[m], dist[m], seg[m], o, span=spans[m],
                              knots=np.asarray(cv.knots.knots), degree=cv.degree)
        checked += len(m)
    assert checked >= 40_000
    assert ties <= checked // 100
    # the per-curve cell indices the bench builds change no result bit
    assert cset.build_cells(12) > 0
    r = [x.cpu().numpy() for x in cset.project_device(q, cid)]
    for k, ref in ((0, t), (1, foot), (2, dist), (4, seg)):
        assert np.array_equal(r[k], ref), k
