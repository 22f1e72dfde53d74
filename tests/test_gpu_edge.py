"""Non-finite, overflowing and empty inputs through the drop-in API, against the
reference's own outputs (tests/golden/edge.npz, made by make_golden.py from
splinemat.project_prepared): +-inf coordinates, |q| up to 1e300 (|C - q|^2
overflows to inf), interleaved with ordinary queries in one batch.  NaN has
no reference answer (the numba kernel leaves np.empty memory in place); for it
the package returns NaN and must leave the other queries untouched."""
import numpy as np
import pytest

from conftest import load_golden


def _assert_edge_parity(t, foot, dist, z):
    """North-star bars (t within 1e-6, distance 1e-9 relative, foot 1e-6 as in
    test_gpu_project.py), with the non-finite outputs required to be the
    reference's exactly (inf stays inf)."""
    for v, r in ((t, z["t"]), (foot, z["foot"]), (dist, z["dist"])):
        fin = np.isfinite(r)
        assert np.array_equal(np.isfinite(v), fin)
        assert np.array_equal(v[~fin], r[~fin])
    assert np.all(np.abs(t - z["t"]) <= 1e-6)
    assert np.abs(foot - z["foot"]).max() <= 1e-6
    f = np.isfinite(z["dist"])
    assert np.all(np.abs(dist[f] - z["dist"][f]) <= np.maximum(1e-9 * z["dist"][f], 1e-12))


def _prep(z):
    from paper_2504_11498_b200 import BSplineCurve, prepare_curve
    c = BSplineCurve(int(z["degree"]), z["knots"], z["ctrl"])
    return prepare_curve(c, 1e-4)


def test_oracle_matches_reference_edge(oracle_lib):
    """The C oracle reproduces the reference on the same non-finite inputs."""
    from oracle import prep as P
    z = load_golden("edge.npz")
    pr = P.prepare(int(z["degree"]), z["knots"], z["ctrl"], 1e-4)
    o = oracle_lib.project_block(pr["seg_pts"], pr["seg_ta"], pr["seg_tb"], pr["seam_t"],
                                 pr["seam_pt"], z["queries"], workers=2)
    for k in ("t", "foot", "dist", "cand"):
        assert np.array_equal(o[k], z[k]), k


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [{}, {"screen": False}])
def test_nonfinite_queries_match_reference(gpu, mode):
    from paper_2504_11498_b200 import project_prepared
    z = load_golden("edge.npz")
    t, foot, dist, cand = project_prepared(_prep(z), z["queries"], **mode)
    _assert_edge_parity(t, foot, dist, z)
    assert np.array_equal(cand, z["cand"])


@pytest.mark.gpu
def test_nonfinite_queries_screened(gpu):
    """cand="screened" changes only the candidate count."""
    from paper_2504_11498_b200 import project_prepared
    z = load_golden("edge.npz")
    t, foot, dist, cand = project_prepared(_prep(z), z["queries"], cand="screened")
    _assert_edge_parity(t, foot, dist, z)
    assert np.all(cand >= 0)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [{}, {"cand": "screened"}, {"screen": False}])
def test_nan_query_isolated(gpu, mode):
    from paper_2504_11498_b200 import project_prepared
    z = load_golden("edge.npz")
    prep = _prep(z)
    q = z["queries"].copy()
    q[5] = [np.nan, 0.0, 0.0]
    q[17] = [0.3, np.nan, np.nan]
    t, foot, dist, cand = project_prepared(prep, q, **mode)
    assert np.isnan(t[[5, 17]]).all() and np.isnan(dist[[5, 17]]).all()
    keep = np.ones(len(q), bool)
    keep[[5, 17]] = False
    ref = project_prepared(prep, q[keep], **mode)
    for a, b in zip((t, foot, dist, cand), ref):
        assert np.array_equal(a[keep], b)


@pytest.mark.gpu
def test_empty_batch(gpu):
    from paper_2504_11498_b200 import project_prepared
    z = load_golden("edge.npz")
    prep = _prep(z)
    for mode in ({}, {"cand": "screened"}, {"screen": False}):
        out = project_prepared(prep, np.zeros((0, 3)), **mode)
        assert [x.shape for x in out] == [(0,), (0, 3), (0,), (0,)]
        assert out[3].dtype == np.int64


@pytest.mark.gpu
def test_curve_set_nonfinite_queries(gpu):
    """project_batch: each query's (t, foot, dist) equal project_prepared's on
    its own curve -- which equals the reference's (above) -- with the
    non-finite queries spread over the curves."""
    from paper_2504_11498_b200 import BSplineCurve, prepare_curve, project_batch, project_prepared
    from paper_2504_11498_b200.batch import curve_set_from_prepared
    from paper_2504_11498_b200.fixtures import random_clamped_curve
    z = load_golden("edge.npz")
    preps = [_prep(z), prepare_curve(random_clamped_curve(np.random.default_rng(9), 3, 20, 3), 1e-4),
             prepare_curve(BSplineCurve(int(z["degree"]), z["knots"], 10.0 * z["ctrl"]), 1e-4)]
    cset = curve_set_from_prepared(preps)
    q = z["queries"]
    cid = np.arange(len(q)) % 3
    t, foot, dist, _ = project_batch(cset, q, cid)
    for c in range(3):
        m = cid == c
        rt, rf, rd, _ = project_prepared(preps[c], q[m])
        assert np.array_equal(t[m], rt) and np.array_equal(foot[m], rf)
        assert np.array_equal(dist[m], rd)


@pytest.mark.gpu
def test_surface_nonfinite_queries(gpu):
    """Surfaces: an infinite / overflowing / NaN query yields dist inf / NaN
    and leaves the finite queries' answers unchanged."""
    from paper_2504_11498_b200 import prepare_surface, project_surface_prepared
    from paper_2504_11498_b200.fixtures import random_surface
    s = random_surface(np.random.default_rng(4), 3, 3, 8, 8)
    prep = prepare_surface(s)
    rng = np.random.default_rng(5)
    q = rng.random((64, 3))
    bad = {3: [np.inf, 0, 0], 10: [1e300, 1e300, 0], 20: [0, -np.inf, 1], 33: [np.nan, 0, 0]}
    qb = q.copy()
    for i, v in bad.items():
        qb[i] = v
    u, v, foot, dist, patch = project_surface_prepared(prep, qb, return_patches=True)
    assert np.isinf(dist[[3, 10, 20]]).all()
    assert np.isnan(u[33]) and np.isnan(v[33]) and np.isnan(foot[33]).all() and np.isnan(dist[33])
    assert patch[33] == -1
    keep = np.array([i not in bad for i in range(len(q))])
    ref = project_surface_prepared(prep, q[keep], return_patches=True)
    for a, b in zip((u, v, foot, dist, patch), ref):
        assert np.array_equal(a[keep], b)
