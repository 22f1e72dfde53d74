"""Nearest-over-set projection (nearest.py): one table holding the cubics of
several curves with separator records between them.  The distance equals the
minimum of the per-curve project_prepared distances bit for bit; where that
minimum is unique (next curve farther by > 1e-9) the curve, t, foot point and
cubic index are that curve's own result."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _curves(seed, m=5, dim=3):
    from paper_2504_11498_b200 import prepare_curve
    from paper_2504_11498_b200.fixtures import random_clamped_curve
    rng = np.random.default_rng(seed)
    preps = []
    for i in range(m):
        p = int(rng.integers(3, 8))
        c = random_clamped_curve(rng, p, int(rng.integers(p + 2, 40)), dim, uniform_knots=True)
        preps.append(prepare_curve(c, 1e-4))
    return preps


def _check(preps, q, res):
    from paper_2504_11498_b200 import project_prepared
    cid, t, foot, dist, seg = res
    per = [project_prepared(p, q, return_segments=True) for p in preps]
    D = np.stack([r[2] for r in per])
    best = D.min(axis=0)
    assert np.array_equal(dist, best)
    srt = np.sort(D, axis=0)
    uniq = srt[1] > srt[0] + 1e-9 * np.maximum(1.0, srt[0]) if len(preps) > 1 else np.ones(len(q), bool)
    am = D.argmin(axis=0)
    assert uniq.mean() > 0.9
    assert np.array_equal(cid[uniq], am[uniq])
    for c, r in enumerate(per):
        sel = uniq & (am == c)
        assert np.array_equal(t[sel], r[0][sel])
        assert np.array_equal(foot[sel], r[1][sel])
        assert np.array_equal(seg[sel], r[4][sel])


@pytest.mark.parametrize("n", [3000, 70000])
def test_nearest_matches_per_curve_minimum(gpu, n):
    from paper_2504_11498_b200 import prepare_nearest_set, project_nearest
    preps = _curves(5)
    nset = prepare_nearest_set(preps)
    rng = np.random.default_rng(n)
    ends = np.concatenate([np.stack([p.seam_pt[0], p.seam_pt[-1]]) for p in preps])
    q = np.concatenate([rng.uniform(-0.2, 1.2, (n, 3)), ends])
    res = project_nearest(nset, q)
    _check(preps, q, res)
    if n >= 65536:  # the dense batch built a cell index over the merged table
        assert nset.table.cells is not None


def test_nearest_single_curve_equals_project_prepared(gpu):
    from paper_2504_11498_b200 import prepare_nearest_set, project_nearest, project_prepared
    preps = _curves(9, m=1)
    q = np.random.default_rng(1).uniform(0, 1, (2000, 3))
    cid, t, foot, dist, seg = project_nearest(prepare_nearest_set(preps), q)
    r = project_prepared(preps[0], q, return_segments=True)
    assert (cid == 0).all()
    for a, b in zip((t, foot, dist, seg), (r[0], r[1], r[2], r[4])):
        assert np.array_equal(a, b)


def test_nearest_edge_cases(gpu):
    from paper_2504_11498_b200 import DomainError, prepare_nearest_set, project_nearest
    preps = _curves(3, m=2)
    nset = prepare_nearest_set(preps)
    out = project_nearest(nset, np.zeros((0, 3)))
    assert all(len(a) == 0 for a in out)
    with pytest.raises(DomainError):
        project_nearest(nset, np.zeros((3, 2)))
    with pytest.raises(DomainError):
        prepare_nearest_set([])


def test_nearest_planar_curves(gpu):
    """d = 2 tables (separators and seams in the plane)."""
    from paper_2504_11498_b200 import prepare_nearest_set, project_nearest
    preps = _curves(13, m=4, dim=2)
    q = np.random.default_rng(2).uniform(-0.2, 1.2, (5000, 2))
    _check(preps, q, project_nearest(prepare_nearest_set(preps), q))


@pytest.mark.parametrize("dim", [2, 3])
def test_nearest_vs_c_oracle_per_curve_minimum(gpu, oracle_lib, dim):
    """Against the pinned C oracle (brute force per curve, then the minimum
    over curves): distance within 1e-9 relative; curve id exact unless
    another curve is within 2e-12; t within 1e-6 and the cubic index exact
    (outside the oracle's own ties) on the winning curve."""
    from paper_2504_11498_b200 import prepare_nearest_set, project_nearest
    preps = _curves(31 + dim, m=6, dim=dim)
    rng = np.random.default_rng(77)
    q = np.concatenate([rng.uniform(-0.2, 1.2, (4000, dim)),
                        np.concatenate([p.seam_pt[[0, -1]] for p in preps])])
    cid, t, foot, dist, seg = project_nearest(prepare_nearest_set(preps), q)
    outs = [oracle_lib.project_block(p.seg_pts, p.seg_ta, p.seg_tb, p.seam_t, p.seam_pt, q,
                                     workers=8) for p in preps]
    D = np.stack([o["dist"] for o in outs])
    best = D.min(axis=0)
    assert np.all(np.abs(dist - best) <= np.maximum(1e-9 * best, 1e-12))
    srt = np.sort(D, axis=0)
    uniq = srt[1] > srt[0] + 2e-12
    am = D.argmin(axis=0)
    assert np.array_equal(cid[uniq], am[uniq])
    for c, o in enumerate(outs):
        sel = uniq & (am == c)
        assert np.all(np.abs(t[sel] - o["t"][sel]) <= 1e-6)
        clear = sel & (o["tie"] == 0)
        assert np.array_equal(seg[clear], o["seg"][clear])
