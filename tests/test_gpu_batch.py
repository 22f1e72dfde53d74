"""Multi-curve batch projection (mrep_project_batch, BASELINE configs[2]) vs
the reference's per-curve outputs and the single-curve path.

Bars as for one curve (north star): distance within 1e-9 relative,
parameter within 1e-6, winning segment equal to the oracle's; and the batch
path must be BIT-identical to project_prepared on each curve alone (same
kernels, only the scheduling differs).
"""
import numpy as np
import pytest

from conftest import assert_parity, load_golden

pytestmark = pytest.mark.gpu


def golden_curves(g):
    from paper_2504_11498_b200 import BSplineCurve
    out, co = [], 0
    for i in range(len(g["degree"])):
        n = int(g["n_control"][i])
        out.append(BSplineCurve(int(g["degree"][i]), g["knots"][g["knot_ofs"][i]: g["knot_ofs"][i + 1]],
                                g["ctrl"][co: co + n]))
        co += n
    return out


def test_prepare_curve_set_matches_reference(gpu):
    from paper_2504_11498_b200 import prepare_curve_set
    g = load_golden("batch_mixed.npz")
    curves = golden_curves(g)
    cs = prepare_curve_set(curves, 1e-4)
    assert np.array_equal(cs.seg_ofs, g["seg_ofs"])
    assert np.array_equal(cs.seg_ta, g["seg_ta"]) and np.array_equal(cs.seg_tb, g["seg_tb"])
    assert np.abs(cs.seg_pts - g["seg_pts"]).max() <= 1e-12 * np.sqrt(3)
    # set[c] is the PreparedCurve prepare_curve(curves[c]) returns
    from paper_2504_11498_b200 import prepare_curve
    for c in (0, 7, len(curves) - 1):
        one = prepare_curve(curves[c], 1e-4)
        sub = cs[c]
        for f in ("seg_pts", "seg_ta", "seg_tb", "seam_t", "seam_pt"):
            assert np.array_equal(getattr(one, f), getattr(sub, f)), f


def test_project_batch_matches_reference(gpu, oracle_lib):
    from paper_2504_11498_b200 import curve_set_from_prepared, project_batch
    from paper_2504_11498_b200.project import PreparedCurve
    g = load_golden("batch_mixed.npz")
    ofs = g["seg_ofs"]
    preps = []
    for c in range(len(ofs) - 1):
        a, b = ofs[c], ofs[c + 1]
        pts, ta, tb = g["seg_pts"][a:b], g["seg_ta"][a:b], g["seg_tb"][a:b]
        preps.append(PreparedCurve(None, 1e-4, pts, ta, tb, np.concatenate(([ta[0]], tb)),
                                   np.concatenate((pts[:1, 0], pts[:, 3]))))
    cs = curve_set_from_prepared(preps)
    q, cid = g["queries"], g["curve_ids"]
    t, foot, dist, cand, seg = project_batch(cs, q, cid, return_segments=True)
    assert np.all(np.abs(t - g["t"]) <= 1e-6), np.abs(t - g["t"]).max()
    assert np.all(np.abs(dist - g["dist"]) <= np.maximum(1e-9 * g["dist"], 1e-12))
    assert np.abs(foot - g["foot"]).max() <= 1e-6
    for c, pr in enumerate(preps):
        m = cid == c
        o = oracle_lib.project_block(pr.seg_pts, pr.seg_ta, pr.seg_tb, pr.seam_t, pr.seam_pt,
                                     q[m], workers=4)
        assert np.array_equal(seg[m], o["seg"]), c


def _single_vs_batch(cs, q, cid, curves_to_check):
    from paper_2504_11498_b200 import project_prepared
    t, foot, dist, cand, seg = cs.project_host(q, cid)
    for c in curves_to_check:
        m = cid == c
        if not m.any():
            continue
        r = project_prepared(cs[c], q[m], return_segments=True)
        assert np.array_equal(r[0], t[m]), c
        assert np.array_equal(r[1], foot[m]), c
        assert np.array_equal(r[2], dist[m]), c
        assert np.array_equal(r[4], seg[m]), c
    return t, foot, dist, cand, seg


def test_batch_bit_identical_to_single_curve_path(gpu):
    """cfg3-shaped set (mixed degree 3-9, up to 2048 ctrl pts): the scheduler
    changes nothing but the order of work."""
    from paper_2504_11498_b200 import prepare_curve_set
    from paper_2504_11498_b200.fixtures import mixed_curve_batch
    curves = mixed_curve_batch(120, first_seed=500)
    cs = prepare_curve_set(curves)
    rng = np.random.default_rng(9)
    cid = rng.integers(0, len(curves), 12000).astype(np.int32)
    q = rng.uniform(0, 1, (len(cid), 3))
    cnt = cs.segment_counts()
    check = sorted({int(np.argmax(cnt)), int(np.argmin(cnt)), *range(0, 120, 13)})
    t, foot, dist, cand, seg = _single_vs_batch(cs, q, cid, check)
    assert np.all(np.isfinite(t)) and np.all(seg >= 0)
    # device entry agrees with the host pipeline
    import torch
    dt, dfoot, dd, dc, ds = cs.project_device(torch.from_numpy(q).cuda(),
                                              torch.from_numpy(cid).cuda())
    assert np.array_equal(dt.cpu().numpy(), t) and np.array_equal(ds.cpu().numpy(), seg)
    # both traversal schedules (warp packets / per-lane walks) agree bitwise
    from paper_2504_11498_b200 import _lib as L
    for fl in (L.MREP_PACKET, L.MREP_PER_LANE, L.MREP_GROUP):
        r = cs.project_device(torch.from_numpy(q).cuda(), torch.from_numpy(cid).cuda(),
                              extra_flags=fl)
        for k, ref in ((0, t), (1, foot), (2, dist), (4, seg)):
            assert np.array_equal(r[k].cpu().numpy(), ref), (fl, k)


def test_batch_vs_oracle_brute_force_subsample(gpu, oracle_lib):
    """Brute-force C oracle (the reference kernel) on the GPU-prepared arrays
    of a stratified curve subsample."""
    from paper_2504_11498_b200 import prepare_curve_set, project_batch
    from paper_2504_11498_b200.fixtures import mixed_curve_batch
    curves = mixed_curve_batch(60, first_seed=2000, max_control=600)
    cs = prepare_curve_set(curves)
    rng = np.random.default_rng(10)
    cid = np.repeat(np.arange(len(curves)), 40).astype(np.int32)
    rng.shuffle(cid)
    q = rng.uniform(0, 1, (len(cid), 3))
    t, foot, dist, cand, seg = project_batch(cs, q, cid, return_segments=True)
    for c in range(0, len(curves), 3):
        m = cid == c
        pr = cs[c]
        o = oracle_lib.project_block(pr.seg_pts, pr.seg_ta, pr.seg_tb, pr.seam_t, pr.seam_pt,
                                     q[m], workers=8)
        # t, distance, and the segment EXACT except oracle-detected ties
        assert_parity(t[m], dist[m], seg[m], o)


def test_batch_edge_cases(gpu):
    import torch
    from paper_2504_11498_b200 import DomainError, prepare_curve_set, project_batch
    from paper_2504_11498_b200.fixtures import mixed_curve_batch, single_span_cubic
    cs = prepare_curve_set(mixed_curve_batch(5, max_control=40))
    # empty batch
    out = project_batch(cs, np.zeros((0, 3)), np.zeros(0, np.int32), return_segments=True)
    assert all(len(a) == 0 for a in out)
    # all queries on one curve, and a single query
    q = np.random.default_rng(1).uniform(0, 1, (100, 3))
    a = project_batch(cs, q, np.full(100, 4))
    b = project_batch(cs, q[:1], [4])
    assert a[0][0] == b[0][0]
    with pytest.raises(DomainError):
        project_batch(cs, q[:2], [0, 5])
    # out-of-range ids at the C ABI: NaN outputs and segment -1, others intact
    cid = torch.tensor([0, 99, 1, -3], dtype=torch.int32, device="cuda")
    qd = torch.from_numpy(q[:4]).cuda()
    t, foot, dist, cand, seg = cs.project_device(qd, cid)
    t, seg = t.cpu().numpy(), seg.cpu().numpy()
    assert np.isnan(t[1]) and np.isnan(t[3]) and seg[1] == -1 and seg[3] == -1
    assert np.isfinite(t[0]) and np.isfinite(t[2])
    ref = project_batch(cs, q[[0, 2]], [0, 1])[0]
    assert t[0] == ref[0] and t[2] == ref[1]
    # 2-D set; mixed dimensions rejected
    cs2 = prepare_curve_set([single_span_cubic(2), single_span_cubic(2)])
    r = project_batch(cs2, [[0.5, 0.5], [0.0, 0.0]], [0, 1])
    assert r[2][1] == 0.0
    with pytest.raises(DomainError):
        prepare_curve_set([single_span_cubic(2), single_span_cubic(3)])


def test_curve_set_cells_bitwise_equal_to_walks(gpu):
    """Per-curve cell indices (mrep_curveset_cells_build) are exact: the cell
    scan returns the walks' t / foot / dist / segment bit for bit, including
    queries outside their curve's grid (they walk the tree) and bad ids."""
    import torch
    from paper_2504_11498_b200 import _lib as L, prepare_curve_set
    from paper_2504_11498_b200.fixtures import mixed_curve_batch, single_span_cubic
    curves = mixed_curve_batch(80, first_seed=700, max_control=700)
    cs = prepare_curve_set(curves)
    rng = np.random.default_rng(11)
    cid = rng.integers(0, len(curves), 20000).astype(np.int32)
    q = rng.uniform(0, 1, (len(cid), 3))
    q[::7] = rng.uniform(-1.0, 2.0, (len(q[::7]), 3))  # many outside the grids
    cid[5] = 999
    qd, cd = torch.from_numpy(q).cuda(), torch.from_numpy(cid).cuda()
    ref = [x.cpu().numpy() for x in cs.project_device(qd, cd, extra_flags=L.MREP_GROUP)]
    for gmax in (4, 16):
        nb = cs.build_cells(gmax)
        assert nb > 0
        got = [x.cpu().numpy() for x in cs.project_device(qd, cd)]
        for k in (0, 1, 2, 4):
            assert np.array_equal(got[k], ref[k], equal_nan=True), (gmax, k)
        # forced walks still walk (and agree)
        lane = [x.cpu().numpy() for x in cs.project_device(qd, cd, extra_flags=L.MREP_PER_LANE)]
        assert np.array_equal(lane[2], ref[2], equal_nan=True)
    # a budget too small builds nothing and keeps the old index usable
    assert cs.build_cells(16, max_bytes=1024) == 0
    # host pipeline over an indexed set
    out = cs.project_host(q, np.where(cid == 999, 0, cid))
    assert np.all(np.isfinite(out[0]))
    # 2-D set
    cs2 = prepare_curve_set([single_span_cubic(2), single_span_cubic(2)])
    assert cs2.build_cells(8) > 0
    r = cs2.project_device(torch.tensor([[0.5, 0.5], [0.0, 0.0]], dtype=torch.float64).cuda(),
                           torch.tensor([0, 1], dtype=torch.int32).cuda())
    assert r[2].cpu().numpy()[1] == 0.0
