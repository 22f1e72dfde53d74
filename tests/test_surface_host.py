"""Surface path, CPU side (no GPU): the oracle's decomposition, the
global optimality of its seeded-Newton projection (vs a dense-grid search),
and host-side validation.

The reference has no surface code: the oracle in
oracle/mrep_surface_oracle.c defines the algorithm, and these tests pin it
to independent checks -- Cox-de Boor evaluation for the patches, a dense
global search for the minimiser.
"""
import numpy as np
import pytest


def _surf(pu, pv, n=16, seed=0):
    from paper_2504_11498_b200.fixtures import random_surface
    return random_surface(np.random.default_rng(seed), pu, pv, n, n)


@pytest.mark.parametrize("pu,pv", [(3, 3), (5, 5), (3, 5), (2, 2)])
def test_oracle_patches_evaluate_like_de_boor(pu, pv):
    from oracle import surface as OS
    s = _surf(pu, pv, 12)
    pts, iv = OS.decompose(pu, pv, s.knots_u.knots, s.knots_v.knots, s.control_points)
    assert pts.shape[:2] == (12 - pu, 12 - pv)
    rng = np.random.default_rng(1)
    for _ in range(40):
        i, j = rng.integers(0, pts.shape[0]), rng.integers(0, pts.shape[1])
        a, b = rng.uniform(0, 1, 2)
        S = np.einsum("a,c,acx->x", OS._bern(pu, a), OS._bern(pv, b), pts[i, j])
        u = iv[i, j, 0] + a * (iv[i, j, 1] - iv[i, j, 0])
        v = iv[i, j, 2] + b * (iv[i, j, 3] - iv[i, j, 2])
        T = OS.eval_surface(pu, pv, s.knots_u.knots, s.knots_v.knots, s.control_points,
                            [[u, v]])[0]
        assert np.abs(S - T).max() <= 1e-13


@pytest.mark.parametrize("pu,pv,seed", [(3, 3, 0), (5, 5, 1), (3, 5, 2)])
def test_oracle_minimiser_is_global(oracle_lib, pu, pv, seed):
    from oracle import surface as OS
    s = _surf(pu, pv, 14, seed)
    pts, iv = OS.decompose(pu, pv, s.knots_u.knots, s.knots_v.knots, s.control_points)
    P = pts.reshape(-1, pu + 1, pv + 1, 3)
    rng = np.random.default_rng(10 + seed)
    q = np.concatenate([rng.uniform(0, 1, (24, 3)), rng.uniform(-0.5, 1.5, (6, 3))])
    o = oracle_lib.surface_project(P, iv.reshape(-1, 4), pu, pv, q, workers=8)
    for k in range(len(q)):
        d, _ = OS.dense_truth(P, pu, pv, q[k])
        assert o["dist"][k] <= d * (1 + 1e-9) + 1e-12, (k, o["dist"][k], d)
    # foot is on the surface at the returned parameters
    S = OS.eval_surface(pu, pv, s.knots_u.knots, s.knots_v.knots, s.control_points,
                        np.stack([o["u"], o["v"]], 1))
    assert np.abs(S - o["foot"]).max() <= 1e-12
    assert np.allclose(np.linalg.norm(q - o["foot"], axis=1), o["dist"], rtol=1e-12, atol=1e-14)


def test_oracle_on_surface_points_invert(oracle_lib):
    from oracle import surface as OS
    s = _surf(3, 3, 12, 3)
    pts, iv = OS.decompose(3, 3, s.knots_u.knots, s.knots_v.knots, s.control_points)
    rng = np.random.default_rng(4)
    uv = rng.uniform(0, 1, (30, 2))
    q = OS.eval_surface(3, 3, s.knots_u.knots, s.knots_v.knots, s.control_points, uv)
    o = oracle_lib.surface_project(pts.reshape(-1, 4, 4, 3), iv.reshape(-1, 4), 3, 3, q)
    assert o["dist"].max() <= 1e-12
    assert np.abs(o["u"] - uv[:, 0]).max() <= 1e-8 and np.abs(o["v"] - uv[:, 1]).max() <= 1e-8


def test_validate_surface_errors():
    from paper_2504_11498_b200 import (BSplineSurface, CountMismatch, DomainError,
                                       NonMonotoneKnots, NotClamped, validate_surface)
    s = _surf(3, 3, 8)
    validate_surface(s)
    with pytest.raises(CountMismatch):
        validate_surface(BSplineSurface(3, 3, s.knots_u.knots, s.knots_v.knots,
                                        s.control_points[:-1]))
    bad = np.array(s.knots_u.knots)
    bad[0] = 0.5
    with pytest.raises((NonMonotoneKnots, NotClamped)):
        validate_surface(BSplineSurface(3, 3, bad, s.knots_v.knots, s.control_points))
    with pytest.raises(DomainError):
        validate_surface(BSplineSurface(3, 3, s.knots_u.knots, s.knots_v.knots,
                                        s.control_points[..., :2]))


def test_surface_fixture_shape():
    s = _surf(5, 5, 64)
    assert s.control_points.shape == (64, 64, 3)
    z = s.control_points[..., 2]
    assert z.min() == 0.0 and z.max() == 1.0
    assert s.domain_u == (0.0, 1.0) and s.domain_v == (0.0, 1.0)


def test_surface_oracle_decomposition_pinned_to_reference():
    """The surface oracle's decomposition (oracle/surface.py) equals the
    reference's decompose_to_bezier applied along v, then u (surfdec.npz)."""
    import sys
    import os
    sys.path.insert(0, os.path.dirname(__file__))
    from conftest import load_golden
    from oracle import surface as OS
    z = load_golden("surfdec.npz")
    for name in z["names"]:
        g = lambda k: z[f"{name}_{k}"]  # noqa: E731
        pts, iv = OS.decompose(int(g("pu")), int(g("pv")), g("U"), g("V"), g("P"))
        assert np.array_equal(iv, g("iv"))
        assert np.abs(pts - g("patches")).max() <= 1e-13
