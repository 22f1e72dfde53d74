"""The reference's API-level tests (tests/test_project.py, test_distance.py,
test_acceptance.py criteria 1-5) ported to this package: same inputs, same
assertions, GPU underneath."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ALPHA = 1e-4


def grid_oracle(curve, queries, grid=4096):
    """Dense-grid nearest distance + resolution (test-side check, after
    oracle.py:95-128), on the host with the pinned prep oracle."""
    from oracle import prep as P
    lo, hi = curve.domain
    ts = np.linspace(lo, hi, grid)
    pts = P.eval_curve(curve.degree, curve.knots.knots, curve.control_points, ts)
    res = float(np.linalg.norm(np.diff(pts, axis=0), axis=1).max())
    d = np.sqrt(((queries[:, None, :] - pts[None]) ** 2).sum(-1)).min(1)
    return d, res


class TestProjectPoints:
    def test_query_at_curve_start(self, gpu):
        from paper_2504_11498_b200 import project_points
        from paper_2504_11498_b200.fixtures import single_span_cubic
        c = single_span_cubic()
        r = project_points(c, [c.control_points[0]])[0]
        assert r.t_star == 0.0 and r.distance == 0.0

    def test_on_curve_point_within_tolerance(self, gpu):
        from paper_2504_11498_b200 import eval_de_boor, project_points
        from paper_2504_11498_b200.fixtures import single_span_cubic
        c = single_span_cubic()
        r = project_points(c, [eval_de_boor(c, 0.3)], tolerance=1e-4)[0]
        assert r.distance <= 1e-4

    def test_foot_matches_curve(self, gpu):
        from paper_2504_11498_b200 import eval_de_boor, project_points
        from paper_2504_11498_b200.fixtures import random_clamped_curve, random_queries
        rng = np.random.default_rng(10)
        c = random_clamped_curve(rng, 5, 12, 3)
        for r in project_points(c, random_queries(rng, 20, 3)):
            assert np.linalg.norm(r.foot - eval_de_boor(c, r.t_star)) <= 2e-4

    def test_kernel_matches_per_op_route(self, gpu):
        from paper_2504_11498_b200 import prepare_curve, project_prepared
        from paper_2504_11498_b200.fixtures import random_clamped_curve, random_queries
        from paper_2504_11498_b200.project import project_single_reference
        rng = np.random.default_rng(11)
        c = random_clamped_curve(rng, 4, 10, 2)
        prep = prepare_curve(c, 1e-4)
        qs = random_queries(rng, 40, 2)
        t, foot, dist, cand = project_prepared(prep, qs, screen=False)
        for i, q in enumerate(qs):
            ref = project_single_reference(prep, q)
            assert abs(dist[i] - ref.distance) <= 1e-10
            assert abs(t[i] - ref.t_star) <= 2e-6
            assert cand[i] == ref.candidates_examined

    def test_deterministic_across_workers(self, gpu):
        from paper_2504_11498_b200 import prepare_curve, project_prepared
        from paper_2504_11498_b200.fixtures import random_clamped_curve, random_queries
        rng = np.random.default_rng(12)
        prep = prepare_curve(random_clamped_curve(rng, 5, 14, 3), 1e-4)
        qs = random_queries(rng, 300, 3)
        outs = [project_prepared(prep, qs, workers=w) for w in (1, 2, 8)]
        for o in outs[1:]:
            for a, b in zip(outs[0], o):
                assert np.array_equal(a, b)

    def test_dimension_mismatch(self, gpu):
        from paper_2504_11498_b200 import DomainError, project_points
        from paper_2504_11498_b200.fixtures import single_span_cubic
        with pytest.raises(DomainError):
            project_points(single_span_cubic(), np.zeros((3, 3)))

    def test_elimination_soundness(self, gpu):
        from paper_2504_11498_b200 import prepare_curve, project_prepared
        from paper_2504_11498_b200.fixtures import random_clamped_curve, random_queries
        rng = np.random.default_rng(13)
        prep = prepare_curve(random_clamped_curve(rng, 5, 12, 2), 1e-4)
        qs = random_queries(rng, 100, 2)
        t, foot, dist, cand, stats, sound = project_prepared(prep, qs, with_stats=True,
                                                             soundness_samples=64)
        m = np.isfinite(sound)
        assert np.all(sound[m] >= dist[m] ** 2 - 1e-10)


class TestEdgeCases:
    def test_c0_kink(self, gpu):
        from paper_2504_11498_b200 import BSplineCurve, project_points
        curve = BSplineCurve(3, [0, 0, 0, 0, 0.5, 0.5, 0.5, 1, 1, 1, 1],
                             [[0.0, 0.0], [0.4, 0.8], [0.8, 1.0], [1.0, 0.5], [1.2, 1.0],
                              [1.6, 0.8], [2.0, 0.0]])
        rng = np.random.default_rng(20)
        qs = np.concatenate([rng.uniform([0, 0], [2, 1.2], (40, 2)), [[1.0, 0.0], [1.0, 1.5]]])
        res = project_points(curve, qs, tolerance=1e-4)
        od, r = grid_oracle(curve, qs)
        for x, o in zip(res, od):
            assert abs(x.distance - o) <= 1e-4 + r

    def test_degree_one_polyline(self, gpu):
        from paper_2504_11498_b200 import BSplineCurve, project_points
        curve = BSplineCurve(1, [0, 0, 0.3, 0.7, 1, 1],
                             [[0.0, 0.0], [1.0, 1.0], [2.0, 0.5], [3.0, 1.5]])
        qs = np.random.default_rng(21).uniform([0, -0.5], [3, 2.0], (30, 2))
        res = project_points(curve, qs, tolerance=1e-4)
        od, r = grid_oracle(curve, qs)
        for x, o in zip(res, od):
            assert abs(x.distance - o) <= 1e-4 + r

    def test_non_unit_domain(self, gpu):
        from paper_2504_11498_b200 import BSplineCurve, project_points
        from paper_2504_11498_b200.fixtures import random_clamped_curve, random_queries
        rng = np.random.default_rng(22)
        base = random_clamped_curve(rng, 4, 9, 2)
        scaled = BSplineCurve(4, 2.0 + 10.0 * base.knots.knots, base.control_points)
        qs = random_queries(rng, 30, 2)
        for a, b in zip(project_points(base, qs), project_points(scaled, qs)):
            assert abs((2.0 + 10.0 * a.t_star) - b.t_star) <= 1e-4
            assert abs(a.distance - b.distance) <= 1e-9


class TestInvert:
    def test_endpoints_exact(self, gpu):
        from paper_2504_11498_b200 import eval_de_boor, invert_point
        from paper_2504_11498_b200.fixtures import random_clamped_curve
        c = random_clamped_curve(np.random.default_rng(14), 4, 9, 3)
        lo, hi = c.domain
        assert invert_point(c, eval_de_boor(c, lo)) == lo
        assert invert_point(c, eval_de_boor(c, hi)) == hi

    def test_random_points(self, gpu):
        from paper_2504_11498_b200 import eval_de_boor, invert_point
        from paper_2504_11498_b200.fixtures import random_clamped_curve
        rng = np.random.default_rng(15)
        c = random_clamped_curve(rng, 5, 12, 2)
        lo, hi = c.domain
        for _ in range(20):
            t = rng.uniform(lo, hi)
            assert abs(invert_point(c, eval_de_boor(c, t)) - t) <= 5e-4

    def test_off_curve_rejected(self, gpu):
        from paper_2504_11498_b200 import PointNotOnCurve, invert_point
        from paper_2504_11498_b200.fixtures import single_span_cubic
        with pytest.raises(PointNotOnCurve):
            invert_point(single_span_cubic(), np.array([5.0, 5.0]))


class TestPerOp:
    def test_collinear_ramp_hull(self, gpu):
        from paper_2504_11498_b200 import NonParametricBezier, hull_x_intersections
        z = hull_x_intersections(NonParametricBezier([-1, -0.6, -0.2, 0.2, 0.6, 1.0]))
        assert abs(z[0] - 0.5) <= 1e-14 and abs(z[1] - 0.5) <= 1e-14
        assert hull_x_intersections(NonParametricBezier([1.0] * 6)) is None

    def test_clip_root_linear_and_quintic(self, gpu):
        from paper_2504_11498_b200 import NonParametricBezier, NoRoot, Poly, clip_root, rebase
        res = clip_root(NonParametricBezier(np.arange(6) / 5.0 - 0.3))
        assert res.iterations == 1 and abs(res.root - 0.3) <= 1e-12
        coeffs = np.polynomial.polynomial.polyfromroots([0.7, -1.0, -2.0, 3.0, 4.0])
        b = rebase(Poly(coeffs))
        if not (b.e_start < 0 <= b.e_end):
            b = rebase(Poly(-coeffs))
        r = clip_root(b)
        assert abs(r.root - 0.7) <= 1e-6 and r.converged_at is not None and r.converged_at <= 3
        with pytest.raises(NoRoot):
            clip_root(NonParametricBezier([1.0, 2.0, 1.5, 2.5, 1.0, 0.5]))

    def test_clip_and_rebase(self, gpu):
        from paper_2504_11498_b200 import NonParametricBezier, Poly, clip, rebase
        from paper_2504_11498_b200.basis import subdivision_matrices
        rng = np.random.default_rng(5)
        b = NonParametricBezier(rng.normal(size=6))
        SL, _ = subdivision_matrices(0.4, 5)
        assert np.allclose(clip(b, 0.0, 0.4).ordinates, SL @ b.ordinates, atol=1e-14)
        out = clip(b, 0.2, 0.6)
        for u in np.linspace(0, 1, 7):
            assert abs(out(u) - b(0.2 + 0.4 * u)) <= 1e-12
        a = rng.normal(size=6)
        r = rebase(Poly(a))
        assert abs(r.e_start - a[0]) <= 1e-14 and abs(r.e_end - a.sum()) <= 1e-12

    def test_solve_quartic_and_split(self, gpu):
        from paper_2504_11498_b200 import (CubicApproxSegment, distance_polys, monotonic_split,
                                           solve_quartic)
        roots = solve_quartic(np.polynomial.polynomial.polyfromroots([0.2, 0.5, 0.9, 3.0]))
        assert np.allclose(roots, [0.2, 0.5, 0.9], atol=1e-10)
        r2 = solve_quartic(np.polynomial.polynomial.polyfromroots([1.5, 2.5, -7, 9]), (1.0, 3.0))
        assert np.allclose(r2, [1.5, 2.5], atol=1e-9)
        rng = np.random.default_rng(3)
        seg = CubicApproxSegment(rng.uniform(0, 1, (4, 3)), (0.0, 1.0), 0.0)
        q = rng.uniform(0, 1, 3)
        pieces = monotonic_split(seg, q)
        assert pieces[0].source_interval[0] == 0.0 and pieces[-1].source_interval[1] == 1.0
        e = distance_polys(seg, q).e
        assert abs(e(0.0) - 2 * (seg.control_points[0] - q) @ (3 * (seg.control_points[1] - seg.control_points[0]))) <= 1e-12


class TestAcceptance:
    def test_criterion_1_decomposition_exactness(self, gpu):
        from oracle import prep as P
        from paper_2504_11498_b200 import decompose_to_bezier, eval_de_boor_many
        from paper_2504_11498_b200.fixtures import random_clamped_curve
        rng = np.random.default_rng(101)
        worst = 0.0
        for i in range(60):
            deg = int(rng.integers(2, 9))
            n = int(rng.integers(max(deg + 1, 5), 51))
            c = random_clamped_curve(rng, deg, n, 2 if i % 2 == 0 else 3, smooth=bool(i % 3))
            dg = float(np.linalg.norm(c.control_points.max(0) - c.control_points.min(0)))
            segs = decompose_to_bezier(c)
            lo, hi = c.domain
            ts = np.linspace(lo, hi, 256)
            ref = eval_de_boor_many(c, ts)
            for s in segs:
                ta, tb = s.source_interval
                m = (ts >= ta) & (ts <= tb)
                if m.any():
                    dev = np.linalg.norm(s.evaluate((ts[m] - ta) / (tb - ta)) - ref[m], axis=1).max()
                    worst = max(worst, dev / dg)
        assert worst <= 1e-9

    def test_criterion_2_tolerance(self, gpu):
        from paper_2504_11498_b200 import (approximate_error_controlled, decompose_to_bezier,
                                           measure_l1_error)
        from paper_2504_11498_b200.fixtures import TABLE_SHAPES, table_shaped_curve
        rng = np.random.default_rng(202)
        worst = 0.0
        for deg, kl in TABLE_SHAPES:
            for dim in (2, 3):
                segs = decompose_to_bezier(table_shaped_curve(rng, deg, kl, dim))
                for cu in approximate_error_controlled(segs, ALPHA):
                    seg = next(s for s in segs if s.source_interval[0] <= cu.source_interval[0]
                               < s.source_interval[1])
                    worst = max(worst, measure_l1_error(cu, seg, samples=1024)[0])
        assert worst <= ALPHA

    def test_criterion_3_inversion(self, gpu):
        from paper_2504_11498_b200 import eval_de_boor_many, prepare_curve, project_prepared
        from paper_2504_11498_b200.fixtures import random_clamped_curve
        rng = np.random.default_rng(303)
        worst, ends = 0.0, []
        for i in range(20):
            deg = int(rng.integers(4, 7))
            c = random_clamped_curve(rng, deg, int(rng.integers(deg + 2, 16)), 2 if i % 2 == 0 else 3)
            prep = prepare_curve(c, ALPHA)
            lo, hi = c.domain
            tt = rng.uniform(lo, hi, 50)
            t, _, _, _ = project_prepared(prep, eval_de_boor_many(c, tt))
            worst = max(worst, float(np.abs(t - tt).max()))
            te = project_prepared(prep, eval_de_boor_many(c, [lo, hi]))[0]
            ends += [abs(te[0] - lo), abs(te[1] - hi)]
        assert worst <= 5e-4 and max(ends) == 0.0

    def test_criterion_4_5_optimality_and_clipping(self, gpu):
        from paper_2504_11498_b200 import prepare_curve, project_prepared
        from paper_2504_11498_b200.fixtures import random_clamped_curve, random_queries
        rng = np.random.default_rng(20240)
        pieces = c3 = cf = 0
        for i in range(10):
            deg = int(rng.integers(4, 7))
            dim = 2 if i % 2 == 0 else 3
            c = random_clamped_curve(rng, deg, int(rng.integers(deg + 2, 18)), dim)
            prep = prepare_curve(c, ALPHA)
            qs = random_queries(rng, 1000, dim)
            t, foot, dist, cand, stats, sound = project_prepared(prep, qs, with_stats=True,
                                                                 soundness_samples=64)
            od, res = grid_oracle(c, qs)
            assert np.all(np.abs(dist - od) <= ALPHA + res)
            fin = np.isfinite(sound)
            assert np.all(sound[fin] >= dist[fin] ** 2 - 1e-10)
            pieces += stats.pieces
            c3 += stats.conv3_source
            cf += stats.conv_final_source
        assert c3 / pieces >= 0.95 and cf == pieces


class TestKnotSpans:
    """Knot span of t* (north star: bit-exact): searchsorted(knots, t*,
    'right') - 1 clipped to [p, n-1], the convention of core.py:108-112."""

    @pytest.mark.parametrize("name", ["cfg1_random", "cfg2", "kink", "deg9", "deg5_2d"])
    def test_spans_of_reference_t(self, gpu, name):
        import sys
        sys.path.insert(0, __import__("os").path.dirname(__file__))
        from conftest import load_golden, oracle_spans
        from paper_2504_11498_b200 import BSplineCurve, PreparedCurve, project_prepared
        z = load_golden(f"project_{name}.npz")
        curve = BSplineCurve(int(z["degree"]), z["knots"], z["ctrl"])
        # the reference's own prepared arrays, so t* is comparable bit for bit
        prep = PreparedCurve.from_arrays(curve, float(z["tolerance"]), z["seg_pts"], z["seg_ta"],
                                         z["seg_tb"], z["seam_t"], z["seam_pt"])
        for kw in ({}, {"with_stats": True}):
            out = project_prepared(prep, z["queries"], return_spans=True, **kw)
            t, span = out[0], out[-1]
            assert span.dtype == np.int32
            assert np.array_equal(span, oracle_spans(z["knots"], int(z["degree"]), t))
            straddle = span != oracle_spans(z["knots"], int(z["degree"]), z["t"])
            assert not straddle.any()
        # the spans of the reference's own t through the device kernel
        assert np.array_equal(prep.knot_spans(z["t"]),
                              oracle_spans(z["knots"], int(z["degree"]), z["t"]))

    def test_span_edges(self, gpu):
        from paper_2504_11498_b200 import BSplineCurve, PreparedCurve
        knots = np.array([0, 0, 0, 0, 0.25, 0.5, 0.5, 0.75, 1, 1, 1, 1], dtype=float)
        curve = BSplineCurve(3, knots, np.random.default_rng(0).uniform(0, 1, (8, 3)))
        prep = PreparedCurve(curve, 1e-4, np.zeros((1, 4, 3)), [0.0], [1.0], [0.0, 1.0],
                             np.zeros((2, 3)))
        t = np.array([0.0, 0.1, 0.25, 0.4999999999, 0.5, 0.74, 0.75, 0.999, 1.0])
        want = [3, 3, 4, 4, 6, 6, 7, 7, 7]
        assert prep.knot_spans(t).tolist() == want

    def test_batch_spans(self, gpu):
        import sys
        sys.path.insert(0, __import__("os").path.dirname(__file__))
        from conftest import oracle_spans
        from paper_2504_11498_b200 import prepare_curve_set, project_batch
        from paper_2504_11498_b200.fixtures import mixed_curve_batch
        curves = mixed_curve_batch(12, max_control=300)
        cs = prepare_curve_set(curves)
        rng = np.random.default_rng(4)
        cid = rng.integers(0, 12, 3000)
        q = rng.uniform(0, 1, (3000, 3))
        t, foot, dist, cand, seg, span = project_batch(cs, q, cid, return_segments=True,
                                                       return_spans=True)
        for c in range(12):
            m = cid == c
            cv = curves[c]
            assert np.array_equal(span[m], oracle_spans(cv.knots.knots, cv.degree, t[m]))
