"""Surface projection on the B200 (mrep_surface.cu) vs the C oracle
(oracle/mrep_surface_oracle.c, the same algorithm by brute force).

Bars (the north star's, applied to surfaces): distance within 1e-9 relative
(absolute floor 1e-12), parameters within 1e-6 where the minimiser is
unique, winning patch equal (>= 99.9%; exact ties go to the smaller id).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _surf(pu, pv, n, seed=0):
    from paper_2504_11498_b200.fixtures import random_surface
    return random_surface(np.random.default_rng(seed), pu, pv, n, n)


@pytest.mark.parametrize("pu,pv", [(3, 3), (5, 5), (3, 5), (1, 1)])
def test_decompose_surface_matches_oracle(gpu, pu, pv):
    from oracle import surface as OS
    from paper_2504_11498_b200 import decompose_surface, prepare_surface
    s = _surf(pu, pv, 20)
    pts, iv = OS.decompose(pu, pv, s.knots_u.knots, s.knots_v.knots, s.control_points)
    prep = prepare_surface(s)
    assert prep.patch_pts.shape == pts.shape
    assert np.array_equal(prep.patch_iv, iv)
    assert np.abs(prep.patch_pts - pts).max() <= 1e-12
    patches = decompose_surface(s)
    assert len(patches) == pts.shape[0] * pts.shape[1]
    assert patches[5].source_rect == ((iv.reshape(-1, 4)[5, 0], iv.reshape(-1, 4)[5, 1]),
                                      (iv.reshape(-1, 4)[5, 2], iv.reshape(-1, 4)[5, 3]))


def test_eval_surface_matches_oracle(gpu):
    from oracle import surface as OS
    from paper_2504_11498_b200 import eval_surface
    s = _surf(3, 5, 15)
    uv = np.random.default_rng(2).uniform(0, 1, (200, 2))
    uv[:4] = [[0, 0], [1, 1], [0, 1], [1, 0]]
    a = eval_surface(s, uv)
    b = OS.eval_surface(3, 5, s.knots_u.knots, s.knots_v.knots, s.control_points, uv)
    assert np.abs(a - b).max() <= 1e-13


def _check(gpu_out, o):
    u, v, foot, dist, patch = gpu_out
    assert np.all(np.abs(dist - o["dist"]) <= np.maximum(1e-9 * o["dist"], 1e-12)), \
        np.abs(dist - o["dist"]).max()
    same = patch == o["patch"]
    # the patch id EXACT except oracle-detected ties (another patch's minimum
    # within dmin (1 + 1e-9) + 1e-12: a foot on a shared edge)
    bad = np.nonzero(~same & (o["tie"] == 0))[0]
    assert bad.size == 0, f"{bad.size} patch mismatches outside ties, e.g. {bad[:5]}"
    assert np.abs(u[same] - o["u"][same]).max() <= 1e-6
    assert np.abs(v[same] - o["v"][same]).max() <= 1e-6
    assert np.abs(foot[same] - o["foot"][same]).max() <= 1e-6


@pytest.mark.parametrize("pu,pv,n", [(3, 3, 24), (5, 5, 24), (3, 5, 18), (2, 2, 12)])
def test_projection_matches_oracle(gpu, oracle_lib, pu, pv, n):
    from paper_2504_11498_b200 import prepare_surface, project_surface_prepared
    s = _surf(pu, pv, n, seed=pu + pv)
    prep = prepare_surface(s)
    rng = np.random.default_rng(7)
    q = np.concatenate([rng.uniform(0, 1, (1500, 3)), rng.uniform(-1, 2, (300, 3)),
                        s.control_points[[0, -1], [0, -1]]])
    g = project_surface_prepared(prep, q, return_patches=True)
    o = oracle_lib.surface_project(prep.patch_pts.reshape(-1, pu + 1, pv + 1, 3),
                                   prep.patch_iv.reshape(-1, 4), pu, pv, q, workers=16)
    _check(g, o)


def test_unsorted_and_sorted_agree(gpu):
    from paper_2504_11498_b200 import _lib as L, prepare_surface
    s = _surf(3, 3, 32)
    prep = prepare_surface(s)
    q = np.random.default_rng(3).uniform(0, 1, (20000, 3))
    a = prep.table.project(q)
    b = prep.table.project(q, extra_flags=L.MREP_NO_SORT)
    for x, y in zip(a, b):
        assert np.array_equal(x.cpu().numpy(), y.cpu().numpy())


def test_on_surface_points_invert(gpu):
    from paper_2504_11498_b200 import eval_surface, invert_surface_point, prepare_surface
    from paper_2504_11498_b200 import project_surface_prepared, PointNotOnCurve
    s = _surf(3, 3, 20, 5)
    prep = prepare_surface(s)
    uv = np.random.default_rng(4).uniform(0, 1, (2000, 2))
    q = eval_surface(s, uv)
    u, v, foot, dist = project_surface_prepared(prep, q)
    assert dist.max() <= 1e-12
    assert np.abs(u - uv[:, 0]).max() <= 1e-7 and np.abs(v - uv[:, 1]).max() <= 1e-7
    uu, vv = invert_surface_point(s, q[0])
    assert abs(uu - uv[0, 0]) <= 1e-7 and abs(vv - uv[0, 1]) <= 1e-7
    with pytest.raises(PointNotOnCurve):
        invert_surface_point(s, q[0] + np.array([0.0, 0.0, 0.5]))


def test_surface_edge_cases(gpu):
    from paper_2504_11498_b200 import (BSplineSurface, DomainError, prepare_surface,
                                       project_surface_points, project_surface_prepared)
    s = _surf(3, 3, 8)
    prep = prepare_surface(s)
    out = project_surface_prepared(prep, np.zeros((0, 3)), return_patches=True)
    assert all(len(a) == 0 for a in out)
    with pytest.raises(DomainError):
        project_surface_prepared(prep, np.zeros((3, 2)))
    r = project_surface_points(s, [s.control_points[0, 0], [5.0, 5.0, 5.0]])
    assert r[0].distance == 0.0 and r[0].uv == (0.0, 0.0) and r[0].patch == 0
    assert r[1].distance > 0
    with pytest.raises(DomainError):  # unsupported degree pair
        prepare_surface(BSplineSurface(2, 4, s.knots_u.knots[1:-1], np.concatenate(
            ([0.0] * 5, np.linspace(0, 1, 5)[1:-1], [1.0] * 5)), s.control_points[:7, :8]))


def test_large_surface_screened_vs_oracle_subsample(gpu, oracle_lib):
    """cfg4 size (64 x 64 net, 3721 bicubic patches), 2e5 queries; the
    brute-force oracle on a subsample."""
    from paper_2504_11498_b200 import prepare_surface, project_surface_prepared
    s = _surf(3, 3, 64, 11)
    prep = prepare_surface(s)
    q = np.random.default_rng(12).uniform(0, 1, (200000, 3))
    g = project_surface_prepared(prep, q, return_patches=True)
    idx = np.random.default_rng(13).choice(len(q), 300, replace=False)
    o = oracle_lib.surface_project(prep.patch_pts.reshape(-1, 4, 4, 3),
                                   prep.patch_iv.reshape(-1, 4), 3, 3, q[idx], workers=16)
    _check(tuple(a[idx] for a in g), o)


@pytest.mark.parametrize("pu,pv,n,grid", [(3, 3, 24, 16), (3, 3, 24, 64), (5, 5, 14, 32),
                                          (3, 5, 12, 8), (1, 1, 30, 40), (3, 3, 82, 48)])
def test_cell_index_matches_tree_walk(gpu, pu, pv, n, grid):
    """mrep_surface_cells_build + MREP_CELLS: bit-identical to the hierarchy
    walk, for queries inside the grid, outside it and on the surface (the
    82 x 82 net has 6241 patches: the branch-and-bound cell bound)."""
    from paper_2504_11498_b200 import _lib as L, eval_surface, prepare_surface
    s = _surf(pu, pv, n, seed=3 * pu + pv)
    prep = prepare_surface(s)
    tab = prep.table
    rng = np.random.default_rng(grid)
    q = np.concatenate([rng.uniform(0, 1, (30000, 3)), rng.uniform(-0.5, 1.5, (5000, 3)),
                        eval_surface(s, rng.uniform(0, 1, (3000, 2))),
                        s.control_points[[0, -1], [0, -1]]])
    tab.use_cells = False
    a = [x.cpu().numpy() for x in tab.project(q)]
    tab.build_cells(grid)
    b = [x.cpu().numpy() for x in tab.project(q, extra_flags=L.MREP_CELLS)]
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("scale", [1e-22, 1e18])
def test_extreme_scales_use_exact_nets(gpu, oracle_lib, scale):
    """Coordinates far outside float's comfortable range (|S|^2 ~ 1e36 or
    ~1e-44): the Bernstein filter must switch to the double nets instead of
    pruning real patches on an overflowed / denormal float bound."""
    from paper_2504_11498_b200 import BSplineSurface, prepare_surface, project_surface_prepared
    base = _surf(3, 3, 12, 21)
    s = BSplineSurface(3, 3, base.knots_u.knots, base.knots_v.knots,
                       base.control_points * scale)
    prep = prepare_surface(s)
    q = np.random.default_rng(22).uniform(0, 1, (3000, 3)) * scale
    g = project_surface_prepared(prep, q, return_patches=True)
    o = oracle_lib.surface_project(prep.patch_pts.reshape(-1, 4, 4, 3),
                                   prep.patch_iv.reshape(-1, 4), 3, 3, q, workers=16)
    u, v, foot, dist, patch = g
    assert np.all(np.abs(dist - o["dist"]) <= np.maximum(1e-9 * o["dist"], 1e-12 * scale))
    assert np.all((patch == o["patch"]) | (o["tie"] != 0))
