"""GPU decomposition + error-controlled approximation vs the reference.

Bars: identical segment / cubic counts, bit-identical
source intervals, control points within 1e-12 x bbox diagonal (numpy's BLAS
summation order is not reproducible bit-for-bit across machines), measured
errors within 1e-12.
"""
import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def golden_curves():
    from paper_2504_11498_b200 import BSplineCurve
    g = load_golden("prep.npz")
    out = []
    for ci in range(len(g["degree"])):
        d = int(g["dim"][ci])
        out.append(BSplineCurve(int(g["degree"][ci]),
                                g["knots"][g["knot_ofs"][ci]: g["knot_ofs"][ci + 1]],
                                g["ctrl"][g["ctrl_ofs"][ci]: g["ctrl_ofs"][ci + 1], :d]))
    return g, out


def diag(curve):
    cp = curve.control_points
    return float(np.linalg.norm(cp.max(0) - cp.min(0)))


def cp_bound(curve):
    """1e-12 x bbox up to degree 9; high degrees are ill-conditioned (the
    reference's own decomposition bounds are 1e-10 / 1e-7 / 5e-4 at degree
    16 / 24 / 31, tests/test_decompose.py:86-95)."""
    return (1e-12 if curve.degree <= 9 else 1e-9) * max(diag(curve), 1.0)


def test_decompose_matches_reference(gpu):
    from paper_2504_11498_b200 import batched_decompose
    g, curves = golden_curves()
    res = batched_decompose(curves)
    bz = 0
    exact = 0
    for c, segs in zip(curves, res):
        assert not isinstance(segs, Exception)
        for s in segs:
            d = c.dimension
            ref = g["bz_pts"][g["bz_ofs"][bz]: g["bz_ofs"][bz + 1], :d]
            assert tuple(g["bz_iv"][bz]) == s.source_interval
            dev = np.abs(s.control_points - ref).max()
            assert dev <= cp_bound(c), (c.degree, dev)
            exact += np.array_equal(s.control_points, ref)
            bz += 1
    assert bz == len(g["bz_iv"])
    assert exact / bz >= 0.5


def test_decompose_single_matches_batched(gpu):
    from paper_2504_11498_b200 import batched_decompose, decompose_to_bezier
    _, curves = golden_curves()
    one = decompose_to_bezier(curves[3])
    many = batched_decompose(curves)[3]
    for a, b in zip(one, many):
        assert np.array_equal(a.control_points, b.control_points)


def test_approximation_matches_reference(gpu):
    from paper_2504_11498_b200 import approximate_error_controlled, decompose_to_bezier
    g, curves = golden_curves()
    for ci, c in enumerate(curves):
        cubics = approximate_error_controlled(decompose_to_bezier(c), 1e-4)
        sel = np.nonzero(g["cu_curve"] == ci)[0]
        assert len(cubics) == len(sel), (ci, c.degree)
        for k, cu in zip(sel, cubics):
            assert tuple(g["cu_iv"][k]) == cu.source_interval
            assert np.abs(cu.control_points - g["cu_pts"][k][:, : c.dimension]).max() \
                <= cp_bound(c), (ci, c.degree)
            assert abs(cu.measured_error - g["cu_err"][k]) <= 1e-12


def test_prepare_curve_tables_match(gpu):
    from paper_2504_11498_b200 import BSplineCurve, prepare_curve
    for name in ("cfg1_random", "cfg2", "table_n", "kink", "polyline", "deg9", "scaled"):
        z = load_golden(f"project_{name}.npz")
        c = BSplineCurve(int(z["degree"]), z["knots"], z["ctrl"])
        prep = prepare_curve(c, float(z["tolerance"]))
        assert prep.seg_pts.shape == z["seg_pts"].shape, name
        assert np.array_equal(prep.seg_ta, z["seg_ta"]) and np.array_equal(prep.seg_tb, z["seg_tb"])
        assert np.abs(prep.seg_pts - z["seg_pts"]).max() <= 1e-12 * max(diag(c), 1.0)


def test_end_to_end_projection_matches_reference(gpu):
    """prepare_curve + project_prepared (GPU only) vs the reference outputs."""
    from paper_2504_11498_b200 import BSplineCurve, prepare_curve, project_prepared
    for name in ("cfg1_invert", "cfg1_random", "cfg2", "table_n", "deg5_2d", "kink"):
        z = load_golden(f"project_{name}.npz")
        c = BSplineCurve(int(z["degree"]), z["knots"], z["ctrl"])
        prep = prepare_curve(c, float(z["tolerance"]))
        t, foot, dist, cand = project_prepared(prep, z["queries"])
        assert np.all(np.abs(t - z["t"]) <= 1e-6), name
        assert np.all(np.abs(dist - z["dist"]) <= np.maximum(1e-9 * z["dist"], 1e-12)), name
        t2, _, d2, c2, stats, sound = project_prepared(prep, z["queries"], with_stats=True,
                                                       soundness_samples=int(z["soundness"]))
        assert np.mean(c2 == z["cand"]) >= 0.999
        assert np.array_equal(t2, t) and np.array_equal(d2, dist)


def test_batched_decompose_isolates_failures(gpu):
    from paper_2504_11498_b200 import BSplineCurve, GeometryError, batched_decompose
    from paper_2504_11498_b200.fixtures import random_clamped_curve
    rng = np.random.default_rng(5)
    good = [random_clamped_curve(rng, 3, 8, 2) for _ in range(3)]
    bad = BSplineCurve(3, [0, 0, 0, 1, 1, 1, 1], np.zeros((3, 2)))
    res = batched_decompose([good[0], bad, good[1], good[2]], workers=4)
    assert isinstance(res[1], GeometryError)
    assert all(isinstance(r, list) and r for r in (res[0], res[2], res[3]))


def test_levels_and_batch_cap(gpu):
    from paper_2504_11498_b200 import approximate_error_controlled, decompose_to_bezier
    from paper_2504_11498_b200.fixtures import table_shaped_curve
    rng = np.random.default_rng(24)
    segs = decompose_to_bezier(table_shaped_curve(rng, 6, 22, 3))
    out, levels = approximate_error_controlled(segs, 1e-4, collect_levels=True)
    assert levels
    for lv in levels:
        ps = lv.child_prefix_sum
        assert np.all(np.diff(ps) >= 2) and len(ps) == len(lv.compaction_keys) + 1
        assert np.all(lv.compaction_keys < len(lv.segments))
    rng = np.random.default_rng(25)
    segs = decompose_to_bezier(table_shaped_curve(rng, 4, 14, 2))
    a = approximate_error_controlled(segs, 1e-4, batch_cap=4096)
    b = approximate_error_controlled(segs, 1e-4, batch_cap=1)
    assert len(a) == len(b)
    for ca, cb in zip(a, b):
        assert np.array_equal(ca.control_points, cb.control_points)


def test_depth_exceeded(gpu):
    from paper_2504_11498_b200 import DepthExceeded, approximate_error_controlled, decompose_to_bezier
    from paper_2504_11498_b200.fixtures import table_shaped_curve
    segs = decompose_to_bezier(table_shaped_curve(np.random.default_rng(26), 5, 12, 2))
    with pytest.raises(DepthExceeded):
        approximate_error_controlled(segs, 1e-13, max_depth=1)


def test_single_item_ops_vs_oracle(gpu):
    from oracle import prep as P
    from paper_2504_11498_b200 import (BezierSegment, CubicApproxSegment, elevate_degree,
                                       eval_bezier, measure_l1_error, subdivide_and_modify)
    from paper_2504_11498_b200.basis import symbolic_basis_matrix
    from paper_2504_11498_b200.reduce_approx import reduce_points_g1
    rng = np.random.default_rng(808)
    for i in range(40):
        p = 4 + i % 5
        Q = rng.uniform(0, 1, (p + 1, 2 + i % 2))
        sol = reduce_points_g1(Q)
        R, d0, d1 = P.g1_cubic(Q)
        assert abs(sol.delta0 - d0) <= 1e-12 * max(1, abs(d0))
        assert abs(sol.delta1 - d1) <= 1e-12 * max(1, abs(d1))
        assert np.abs(sol.cubic - R).max() <= 1e-13
        assert abs(sol.l2_error - P.l2_error(Q, R)) <= 1e-12
        us = rng.uniform(0, 1, 9)
        assert np.array_equal(eval_bezier(Q, us), np.stack([P.de_casteljau(Q, u) for u in us]))
    seg = BezierSegment(2, rng.uniform(0, 1, (3, 3)), (0.0, 1.0))
    assert np.array_equal(elevate_degree(seg, 5).control_points, P.elevate(seg.control_points, 5))
    orig = BezierSegment(5, rng.uniform(0, 1, (6, 2)), (0.2, 0.9))
    cub = CubicApproxSegment(P.g1_cubic(orig.control_points)[0], (0.2, 0.9), 0.0)
    mx, args = measure_l1_error(cub, orig, samples=1024)
    mx_o, args_o = P.max_error(cub.control_points, (0.2, 0.9), orig.control_points, (0.2, 0.9), 1024)
    assert abs(mx - mx_o) <= 1e-14 and np.array_equal(args, args_o)
    L, R = subdivide_and_modify(cub, orig, 0.37)
    t_split = 0.2 + 0.37 * 0.7
    pin = P.de_casteljau(orig.control_points, (t_split - 0.2) / 0.7)
    assert np.array_equal(L.control_points[3], pin) and np.array_equal(R.control_points[0], pin)
    SL, SR = P.split_matrices(0.37)
    assert np.abs(L.control_points[:3] - (SL @ cub.control_points)[:3]).max() <= 1e-15
    kn = np.concatenate(([0] * 6, np.sort(rng.uniform(0, 1, 9)), [1] * 6))
    for q in range(5, 14):
        assert np.array_equal(symbolic_basis_matrix(kn, 5, q, kn[q]), P.span_basis(kn, 5, q, kn[q]))


def test_eval_de_boor_vs_oracle(gpu):
    from oracle import prep as P
    from paper_2504_11498_b200 import eval_de_boor_many
    from paper_2504_11498_b200.fixtures import random_clamped_curve
    for p in (1, 3, 7):
        c = random_clamped_curve(np.random.default_rng(p), p, 20, 3)
        ts = np.concatenate([np.linspace(0, 1, 101), c.knots.knots[p: -p]])
        got = eval_de_boor_many(c, ts)
        ref = P.eval_curve(p, c.knots.knots, c.control_points, ts)
        assert np.abs(got - ref).max() <= 1e-14
