"""Generate the golden fixtures from the UNMODIFIED reference package.

Run in the build container only (the reference tree does not exist on the GPU
box); the outputs are committed next to this script:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Every array below is produced by the reference's own public API or its numba
kernels (`splinemat._kernels`, numba lane, the production default), so the
fixtures pin both the C oracle (`oracle/`) and the CUDA path to the reference.
Files:
  quartic.npz    _quartic_roots_01 on random + degenerate + real E' inputs
  ops.npz        _distance_poly, _restrict_ordinates, _hull_cross, _clip_root,
                 _eval_ordinates, _decasteljau_point, T5, B3
  project_*.npz  prepared tables + queries + every _project_block output
  prep.npz       curves -> decompose_to_bezier -> approximate_error_controlled
  batch_mixed.npz  a mixed-degree curve set (BASELINE configs[2] shape, small
                 n): prepare_curve + project_prepared per curve, queries
                 interleaved across curves
  anydeg.npz     the public NonParametricBezier ops (__call__,
                 hull_x_intersections, clip, clip_root) at degrees != 5
  verify.npz     oracle.oracle_project_batch (dense grid + ternary search,
                 oracle.py:95-128) on three curves
  edge.npz       non-finite and huge queries (+-inf, 1e150..1e300) mixed
                 with ordinary ones through project_prepared (NaN is left out:
                 the reference returns uninitialised memory for it)
  surfdec.npz    a tensor-product surface decomposed with the reference's
                 decompose_to_bezier along v (every row), then along u (every
                 column of the row segments) -- pins the surface patches
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import splinemat  # noqa: E402
from splinemat import _kernels  # noqa: E402
from splinemat._accel import USING_NUMBA  # noqa: E402
from splinemat._fixtures import (  # noqa: E402
    random_clamped_curve,
    random_queries,
    single_span_cubic,
    table_shaped_curve,
    two_span_uniform_cubic,
)
from splinemat.basis import bernstein_matrix, power_to_bernstein_matrix  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
assert USING_NUMBA, "fixtures must come from the numba (production) lane"


def quartic_cases():
    rng = np.random.default_rng(606)
    rows = [rng.uniform(-1.0, 1.0, (3000, 5))]
    # degeneracy cascade: tiny / zero leading coefficients
    deg = rng.uniform(-1.0, 1.0, (400, 5))
    deg[:100, 4] = 0.0
    deg[100:200, 4] = 1e-14 * rng.uniform(-1, 1, 100)
    deg[200:300, 3:] = 0.0
    deg[300:350, 2:] = 0.0
    deg[350:400, :] = 0.0
    rows.append(deg)
    # biquadratic (q == 0 after depression): c3 = c1 = 0
    bq = rng.uniform(-1.0, 1.0, (200, 5))
    bq[:, 1] = 0.0
    bq[:, 3] = 0.0
    bq[:, 4] = np.abs(bq[:, 4]) + 0.1
    rows.append(bq)
    # constructed roots inside [0,1] incl. double roots and endpoint roots
    cons = []
    for _ in range(400):
        k = int(rng.integers(1, 5))
        rts = list(rng.uniform(-0.2, 1.2, k))
        if rng.uniform() < 0.3 and k >= 2:
            rts[1] = rts[0]
        if rng.uniform() < 0.1:
            rts[0] = 0.0
        if rng.uniform() < 0.1:
            rts[-1] = 1.0
        c = np.polynomial.polynomial.polyfromroots(rts) * rng.uniform(0.5, 3.0)
        c5 = np.zeros(5)
        c5[: len(c)] = c
        cons.append(c5)
    rows.append(np.array(cons))
    # realistic E' inputs from (query, cubic) pairs
    curve = random_clamped_curve(np.random.default_rng(0), 7, 64, 3, uniform_knots=True)
    prep = splinemat.prepare_curve(curve, 1e-4)
    qs = random_queries(np.random.default_rng(1), 60, 3)
    real = []
    e = np.empty(6)
    for q in qs:
        for s in range(prep.seg_pts.shape[0]):
            _kernels._distance_poly(prep.seg_pts[s], q, e)
            real.append(e[1:] * np.arange(1, 6))
    rows.append(np.array(real))
    return np.ascontiguousarray(np.concatenate(rows))


def make_quartic():
    coeffs = quartic_cases()
    n = len(coeffs)
    roots = np.full((n, 4), np.nan)
    counts = np.zeros(n, dtype=np.int64)
    _kernels._quartic_block(coeffs, roots, counts)
    nroots = np.full((n, 4), np.nan)
    ncounts = np.zeros(n, dtype=np.int64)
    _kernels._newton_quartic_block(coeffs, nroots, ncounts)
    np.savez_compressed(os.path.join(OUT, "quartic.npz"), coeffs=coeffs,
                        roots=roots, counts=counts, newton_roots=nroots,
                        newton_counts=ncounts)
    print("quartic", n, "cases; root-count histogram", np.bincount(counts))


def make_ops():
    rng = np.random.default_rng(77)
    m = 2000
    # distance polynomial
    P = rng.uniform(-1, 2, (m, 4, 3))
    Q = rng.uniform(-1, 2, (m, 3))
    E = np.empty((m, 6))
    for i in range(m):
        _kernels._distance_poly(P[i], Q[i], E[i])
    P2 = rng.uniform(-1, 2, (200, 4, 2))
    Q2 = rng.uniform(-1, 2, (200, 2))
    E2 = np.empty((200, 6))
    for i in range(200):
        _kernels._distance_poly(P2[i], Q2[i], E2[i])
    # restriction to [lo, hi]
    B = rng.normal(size=(m, 6))
    lo = rng.uniform(0, 1, m)
    hi = rng.uniform(0, 1, m)
    lo, hi = np.minimum(lo, hi), np.maximum(lo, hi)
    lo[:200] = 0.0
    hi[200:400] = 1.0
    R = np.empty((m, 6))
    for i in range(m):
        R[i] = _kernels._restrict_ordinates(B[i], lo[i], hi[i])
    # hull crossing: random, one-signed, with exact zeros, collinear
    H = rng.normal(size=(m, 6))
    H[:100] = np.abs(H[:100])
    H[100:200, rng.integers(0, 6, 100)] = 0.0
    H[200:250] = np.linspace(-1, 1, 6)[None, :] * rng.uniform(0.1, 2, (50, 1))
    H[250:300, 0] = 0.0
    H[300:350, 5] = 0.0
    hf = np.zeros(m, dtype=np.int64)
    hz = np.zeros((m, 2))
    for i in range(m):
        f, z1, z2 = _kernels._hull_cross(H[i])
        hf[i] = int(f)
        hz[i] = (z1, z2)
    # clipping on eliminated-piece-like ordinates (E(0) < 0 <= E(1))
    C = np.empty((m, 6))
    k = 0
    while k < m:
        b = rng.normal(size=6)
        if b[0] < 0.0 <= b[5] or k % 7 == 0:
            C[k] = b
            k += 1
    tols = np.where(np.arange(m) % 5 == 0, 1e-9, 1e-6)
    iters = np.where(np.arange(m) % 11 == 0, 3, 8)
    croot = np.zeros(m)
    cok = np.zeros(m, dtype=np.int64)
    cused = np.zeros(m, dtype=np.int64)
    cw = np.full((m, 8), np.nan)
    for i in range(m):
        w = np.empty(int(iters[i]))
        r, ok, used = _kernels._clip_root(C[i], tols[i], int(iters[i]), w)
        croot[i], cok[i], cused[i] = r, int(ok), used
        cw[i, : len(w)] = w
    # ordinate evaluation and cubic point evaluation
    U = rng.uniform(0, 1, m)
    EV = np.array([_kernels._eval_ordinates(B[i], U[i]) for i in range(m)])
    DP = np.empty((m, 3))
    for i in range(m):
        _kernels._decasteljau_point(P[i], U[i], DP[i])
    np.savez_compressed(
        os.path.join(OUT, "ops.npz"),
        dp_P=P, dp_q=Q, dp_e=E, dp_P2=P2, dp_q2=Q2, dp_e2=E2,
        rs_b=B, rs_lo=lo, rs_hi=hi, rs_out=R,
        hull_b=H, hull_found=hf, hull_z=hz,
        clip_b=C, clip_tol=tols, clip_iters=iters, clip_root=croot,
        clip_ok=cok, clip_used=cused, clip_widths=cw,
        ev_u=U, ev_out=EV, pt_out=DP,
        T5=np.array(power_to_bernstein_matrix(5)), B3=np.array(bernstein_matrix(3)))
    print("ops", m)


def project_case(name, curve, queries, soundness=16, tol=1e-4, clip_tol=1e-6,
                 max_iter=8):
    prep = splinemat.prepare_curve(curve, tol)
    t, foot, dist, cand, stats, sound = splinemat.project_prepared(
        prep, queries, workers=1, clip_tol=clip_tol, max_iterations=max_iter,
        with_stats=True, soundness_samples=soundness)
    # per-query stats columns (project_prepared only returns totals)
    n = len(queries)
    st = np.zeros((n, 6), dtype=np.int64)
    o = (np.empty(n), np.empty((n, curve.dimension)), np.empty(n),
         np.empty(n, dtype=np.int64), st, np.empty(n))
    _kernels._project_block(prep.seg_pts, prep.seg_ta, prep.seg_tb, prep.seam_t,
                            prep.seam_pt, np.ascontiguousarray(queries, dtype=np.float64),
                            clip_tol, max_iter, soundness, *o)
    assert np.array_equal(o[0], t) and np.array_equal(o[2], dist)
    np.savez_compressed(
        os.path.join(OUT, f"project_{name}.npz"),
        degree=curve.degree, knots=np.array(curve.knots.knots),
        ctrl=np.array(curve.control_points), tolerance=tol,
        clip_tol=clip_tol, max_iter=max_iter, soundness=soundness,
        seg_pts=np.array(prep.seg_pts), seg_ta=np.array(prep.seg_ta),
        seg_tb=np.array(prep.seg_tb), seam_t=np.array(prep.seam_t),
        seam_pt=np.array(prep.seam_pt), queries=np.asarray(queries, dtype=np.float64),
        t=t, foot=foot, dist=dist, cand=cand, stats=st, sound=sound)
    print(f"project_{name}: S={prep.seg_pts.shape[0]} n={n} "
          f"pieces={stats.pieces} hull_misses={stats.hull_misses}")


def make_projection():
    # cfg1: p=3, n=64 -> 61 cubics; on-curve (inversion) and random queries
    c1 = random_clamped_curve(np.random.default_rng(0), 3, 64, 3, uniform_knots=True)
    lo, hi = c1.domain
    ts = np.random.default_rng(1).uniform(lo, hi, 1500)
    onc = splinemat.eval_de_boor_many(c1, np.concatenate([[lo, hi], ts]))
    project_case("cfg1_invert", c1, onc, soundness=0)
    project_case("cfg1_random", c1, random_queries(np.random.default_rng(2), 1500, 3))
    # cfg2: p=7, n=512 -> 510 cubics (subset of the 10^6 queries)
    c2 = random_clamped_curve(np.random.default_rng(0), 7, 512, 3, uniform_knots=True)
    project_case("cfg2", c2, random_queries(np.random.default_rng(1), 400, 3), soundness=0)
    # paper table (n) shape, the acceptance 7b curve
    rng = np.random.default_rng(707)
    cn = table_shaped_curve(rng, 5, 18, 3)
    project_case("table_n", cn, random_queries(np.random.default_rng(708), 2000, 3))
    # 2D curve with soundness sampling
    c2d = random_clamped_curve(np.random.default_rng(13), 5, 12, 2)
    project_case("deg5_2d", c2d, random_queries(np.random.default_rng(14), 1500, 2),
                 soundness=64)
    # edge cases: kink, polyline, single span, seams, far queries, start point
    kink = splinemat.BSplineCurve(3, [0, 0, 0, 0, 0.5, 0.5, 0.5, 1, 1, 1, 1],
                                  [[0.0, 0.0], [0.4, 0.8], [0.8, 1.0], [1.0, 0.5],
                                   [1.2, 1.0], [1.6, 0.8], [2.0, 0.0]])
    rng = np.random.default_rng(20)
    qk = np.concatenate([rng.uniform([0, 0], [2, 1.2], (300, 2)),
                         [[1.0, 0.0], [1.0, 1.5], [1.0, 0.5], [0.0, 0.0], [2.0, 0.0]]])
    project_case("kink", kink, qk)
    poly = splinemat.BSplineCurve(1, [0, 0, 0.3, 0.7, 1, 1],
                                  [[0.0, 0.0], [1.0, 1.0], [2.0, 0.5], [3.0, 1.5]])
    project_case("polyline", poly, np.random.default_rng(21).uniform([0, -0.5], [3, 2.0], (300, 2)))
    ss = single_span_cubic(3)
    qs = np.concatenate([ss.control_points, random_queries(np.random.default_rng(3), 200, 3),
                         np.random.default_rng(4).uniform(-50, 50, (50, 3))])
    project_case("single_span", ss, qs)
    tw = two_span_uniform_cubic()
    prep = splinemat.prepare_curve(tw, 1e-4)
    qt = np.concatenate([prep.seam_pt, np.random.default_rng(5).uniform(-0.5, 1.5, (200, 2))])
    project_case("two_span", tw, qt)
    # non-unit domain and high degree
    base = random_clamped_curve(np.random.default_rng(22), 4, 9, 2)
    scaled = splinemat.BSplineCurve(4, 2.0 + 10.0 * base.knots.knots, base.control_points)
    project_case("scaled", scaled, random_queries(np.random.default_rng(23), 300, 2))
    hd = random_clamped_curve(np.random.default_rng(31), 9, 40, 3, uniform_knots=True)
    project_case("deg9", hd, random_queries(np.random.default_rng(32), 400, 3), soundness=0)


def prep_curves():
    curves = []
    rng = np.random.default_rng(202)
    for degree, klen in [(4, 10), (5, 12), (6, 14), (4, 14), (5, 18), (6, 22),
                         (4, 35), (5, 22), (6, 57), (5, 46)]:
        for dim in (2, 3):
            curves.append(table_shaped_curve(rng, degree, klen, dim))
    curves.append(random_clamped_curve(np.random.default_rng(0), 3, 64, 3, uniform_knots=True))
    curves.append(random_clamped_curve(np.random.default_rng(0), 7, 512, 3, uniform_knots=True))
    curves.append(random_clamped_curve(np.random.default_rng(5), 9, 200, 3, uniform_knots=True))
    curves.append(random_clamped_curve(np.random.default_rng(6), 2, 12, 2))
    curves.append(random_clamped_curve(np.random.default_rng(7), 1, 8, 3))
    for p in (8, 12, 16):
        curves.append(random_clamped_curve(np.random.default_rng(p), p, p + 8, 3, smooth=False))
    curves.append(splinemat.BSplineCurve(3, [0, 0, 0, 0, 0.5, 0.5, 0.5, 1, 1, 1, 1],
                                         np.random.default_rng(1).uniform(0, 1, (7, 2))))
    # interior knot multiplicity p on a degree-5 curve (C0 joint, zero spans)
    curves.append(splinemat.BSplineCurve(
        5, [0] * 6 + [0.4] * 5 + [1] * 6, np.random.default_rng(2).uniform(0, 1, (11, 3))))
    return curves


def make_prep():
    curves = prep_curves()
    degs, kofs, knots, cofs, ctrl, dims = [], [0], [], [0], [], []
    bz_ofs, bz_pts, bz_iv, bz_curve = [0], [], [], []
    cu_pts, cu_iv, cu_err, cu_curve = [], [], [], []
    for ci, c in enumerate(curves):
        degs.append(c.degree)
        dims.append(c.dimension)
        knots.append(np.array(c.knots.knots))
        kofs.append(kofs[-1] + len(c.knots.knots))
        cp = np.zeros((c.control_points.shape[0], 3))
        cp[:, : c.dimension] = c.control_points
        ctrl.append(cp)
        cofs.append(cofs[-1] + len(cp))
        segs = splinemat.decompose_to_bezier(c)
        for s in segs:
            pts = np.zeros((s.degree + 1, 3))
            pts[:, : c.dimension] = s.control_points
            bz_pts.append(pts)
            bz_ofs.append(bz_ofs[-1] + len(pts))
            bz_iv.append(s.source_interval)
            bz_curve.append(ci)
        cubics = splinemat.approximate_error_controlled(segs, 1e-4)
        for cu in cubics:
            pts = np.zeros((4, 3))
            pts[:, : c.dimension] = cu.control_points
            cu_pts.append(pts)
            cu_iv.append(cu.source_interval)
            cu_err.append(cu.measured_error)
            cu_curve.append(ci)
    np.savez_compressed(
        os.path.join(OUT, "prep.npz"),
        degree=np.array(degs), dim=np.array(dims), knot_ofs=np.array(kofs),
        knots=np.concatenate(knots), ctrl_ofs=np.array(cofs), ctrl=np.concatenate(ctrl),
        bz_ofs=np.array(bz_ofs), bz_pts=np.concatenate(bz_pts), bz_iv=np.array(bz_iv),
        bz_curve=np.array(bz_curve), cu_pts=np.array(cu_pts), cu_iv=np.array(cu_iv),
        cu_err=np.array(cu_err), cu_curve=np.array(cu_curve), tolerance=1e-4)
    print("prep", len(curves), "curves,", len(bz_iv), "bezier segments,",
          len(cu_iv), "cubics")


def make_batch(n_curves=16, max_control=160, per_curve=48):
    """Curve i: default_rng(i) draws p ~ U{3..9}, n log-uniform on
    [max(8, p+1), max_control], then random_clamped_curve(rng, p, n, 3,
    uniform_knots=True) -- the generator of fixtures.mixed_curve_batch."""
    curves = []
    for i in range(n_curves):
        rng = np.random.default_rng(i)
        p = int(rng.integers(3, 10))
        lo = max(8, p + 1)
        n = int(round(np.exp(rng.uniform(np.log(lo), np.log(max_control)))))
        n = min(max(n, lo), max_control)
        curves.append(random_clamped_curve(rng, p, n, 3, uniform_knots=True))
    rng = np.random.default_rng(4242)
    cid = rng.permutation(np.repeat(np.arange(n_curves), per_curve)).astype(np.int32)
    q = random_queries(rng, len(cid), 3)
    N = len(cid)
    t, foot, dist, cand = np.empty(N), np.empty((N, 3)), np.empty(N), np.empty(N, np.int64)
    seg_pts, seg_ta, seg_tb, seg_ofs = [], [], [], [0]
    for c, cu in enumerate(curves):
        prep = splinemat.prepare_curve(cu, 1e-4)
        m = cid == c
        r = splinemat.project_prepared(prep, q[m], workers=1)
        t[m], foot[m], dist[m], cand[m] = r
        seg_pts.append(np.array(prep.seg_pts))
        seg_ta.append(np.array(prep.seg_ta))
        seg_tb.append(np.array(prep.seg_tb))
        seg_ofs.append(seg_ofs[-1] + len(prep.seg_ta))
    np.savez_compressed(
        os.path.join(OUT, "batch_mixed.npz"),
        degree=np.array([c.degree for c in curves]),
        n_control=np.array([c.control_points.shape[0] for c in curves]),
        knot_ofs=np.concatenate(([0], np.cumsum([len(c.knots.knots) for c in curves]))),
        knots=np.concatenate([np.array(c.knots.knots) for c in curves]),
        ctrl=np.concatenate([np.array(c.control_points) for c in curves]),
        max_control=max_control, seg_pts=np.concatenate(seg_pts), seg_ta=np.concatenate(seg_ta),
        seg_tb=np.concatenate(seg_tb), seg_ofs=np.array(seg_ofs), queries=q, curve_ids=cid,
        t=t, foot=foot, dist=dist, cand=cand)
    print("batch_mixed", n_curves, "curves,", seg_ofs[-1], "cubics,", N, "queries")


def make_anydeg():
    from splinemat.project import (NonParametricBezier, clip, clip_root,
                                   hull_x_intersections)
    rng = np.random.default_rng(404)
    out = {}
    for n in (1, 2, 3, 4, 7, 9, 15):
        m = 300
        B = rng.normal(size=(m, n + 1))
        B[:40] = np.abs(B[:40])                     # one-signed: no crossing
        B[40:60, rng.integers(0, n + 1, 20)] = 0.0  # exact zeros
        U = rng.uniform(0, 1, m)
        lo = rng.uniform(0, 1, m)
        hi = rng.uniform(0, 1, m)
        lo, hi = np.minimum(lo, hi), np.maximum(lo, hi)
        lo[:30] = 0.0
        hi[30:60] = 1.0
        ev = np.array([NonParametricBezier(B[i])(U[i]) for i in range(m)])
        hf = np.zeros(m, dtype=np.int64)
        hz = np.zeros((m, 2))
        for i in range(m):
            r = hull_x_intersections(NonParametricBezier(B[i]))
            if r is not None:
                hf[i] = 1
                hz[i] = r
        cl = np.array([clip(NonParametricBezier(B[i]), lo[i], hi[i]).ordinates
                       for i in range(m)])
        rs = np.array([_kernels._restrict_ordinates(B[i], lo[i], hi[i]) for i in range(m)])
        # clip_root on eliminated-piece-like (increasing through zero) ordinates
        C = np.sort(rng.normal(size=(m, n + 1)), axis=1)
        C[:, 0] = -np.abs(C[:, 0]) - 1e-3
        C[:, -1] = np.abs(C[:, -1]) + 1e-3
        cr = np.zeros(m)
        cw = np.zeros(m)
        ci = np.zeros(m, dtype=np.int64)
        cc = np.zeros(m, dtype=np.int64)
        for i in range(m):
            res = clip_root(NonParametricBezier(C[i]), 1e-6, 8)
            cr[i], cw[i], ci[i] = res.root, res.width, res.iterations
            cc[i] = -1 if res.converged_at is None else res.converged_at
        for k, v in dict(b=B, u=U, lo=lo, hi=hi, ev=ev, hf=hf, hz=hz, clip=cl, restrict=rs,
                         cb=C, croot=cr, cwidth=cw, citer=ci, cconv=cc).items():
            out[f"d{n}_{k}"] = v
    np.savez_compressed(os.path.join(OUT, "anydeg.npz"), degrees=np.array([1, 2, 3, 4, 7, 9, 15]),
                        **out)
    print("anydeg")


def make_verify():
    from splinemat.oracle import oracle_project_batch
    cases = {}
    for name, (seed, p, n, nq, grid) in dict(cfg1=(0, 3, 64, 600, 4096),
                                              deg7=(3, 7, 96, 400, 4096),
                                              coarse=(5, 5, 30, 300, 257)).items():
        rng = np.random.default_rng(seed)
        curve = random_clamped_curve(rng, p, n, 3, uniform_knots=True)
        q = random_queries(np.random.default_rng(seed + 100), nq, 3)
        t, dist, res = oracle_project_batch(curve, q, grid)
        cases.update({f"{name}_degree": p, f"{name}_knots": np.array(curve.knots.knots),
                      f"{name}_ctrl": np.array(curve.control_points), f"{name}_queries": q,
                      f"{name}_grid": grid, f"{name}_t": t, f"{name}_dist": dist,
                      f"{name}_res": res})
    np.savez_compressed(os.path.join(OUT, "verify.npz"), names=np.array(["cfg1", "deg7", "coarse"]),
                        **cases)
    print("verify")


def make_surfdec():
    """Surface patches by the reference's per-direction curve decomposition."""
    from splinemat import BSplineCurve, decompose_to_bezier
    out = {}
    for name, (pu, pv, nu, nv, seed) in dict(bicubic=(3, 3, 12, 10, 1),
                                              mixed=(3, 5, 9, 11, 2),
                                              biquintic=(5, 5, 10, 10, 3)).items():
        rng = np.random.default_rng(seed)
        U = np.concatenate((np.zeros(pu + 1), np.sort(rng.uniform(0.05, 0.95, nu - pu - 1)),
                            np.ones(pu + 1)))
        V = np.concatenate((np.zeros(pv + 1), np.linspace(0, 1, nv - pv + 1)[1:-1],
                            np.ones(pv + 1)))
        P = rng.uniform(0, 1, (nu, nv, 3))
        rows = [decompose_to_bezier(BSplineCurve(pv, V, P[i])) for i in range(nu)]
        nsv = len(rows[0])
        cols = None
        patches = None
        for js in range(nsv):
            for l in range(pv + 1):
                segs = decompose_to_bezier(BSplineCurve(pu, U, np.array(
                    [rows[i][js].control_points[l] for i in range(nu)])))
                if patches is None:
                    patches = np.zeros((len(segs), nsv, pu + 1, pv + 1, 3))
                    ivs = np.zeros((len(segs), nsv, 4))
                for is_, sg in enumerate(segs):
                    patches[is_, js, :, l] = sg.control_points
                    ivs[is_, js] = (*sg.source_interval, *rows[0][js].source_interval)
        out.update({f"{name}_pu": pu, f"{name}_pv": pv, f"{name}_U": U, f"{name}_V": V,
                    f"{name}_P": P, f"{name}_patches": patches, f"{name}_iv": ivs})
    np.savez_compressed(os.path.join(OUT, "surfdec.npz"),
                        names=np.array(["bicubic", "mixed", "biquintic"]), **out)
    print("surfdec")


def make_edge():
    c = random_clamped_curve(np.random.default_rng(5), 3, 12, 3, uniform_knots=True)
    rng = np.random.default_rng(6)
    big = [[np.inf, 0, 0], [-np.inf, 1, 0], [0, 0, np.inf], [np.inf, -np.inf, 0],
           [1e300, 0, 0], [1e200, 0, 0], [1e150, 1e150, 0], [-1e154, 0, 1e154],
           [1e100, 1e100, 1e100], [1e30, 0, 0]]
    q = rng.random((40, 3))
    q[::4] = np.array(big, dtype=np.float64)
    prep = splinemat.prepare_curve(c, 1e-4)
    t, foot, dist, cand = splinemat.project_prepared(prep, q, workers=1)
    np.savez_compressed(os.path.join(OUT, "edge.npz"), degree=c.degree,
                        knots=np.array(c.knots.knots), ctrl=np.array(c.control_points),
                        queries=q, t=t, foot=foot, dist=dist, cand=cand)
    print("edge", t[::4], dist[::4], cand[::4])


if __name__ == "__main__":
    which = sys.argv[1:] or ["quartic", "ops", "projection", "prep", "batch", "anydeg", "verify",
                             "surfdec", "edge"]
    for w in which:
        globals()["make_" + w]()
