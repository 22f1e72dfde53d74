"""Curve-set (BASELINE configs[2]) host logic and oracle pin, no GPU.

* the cfg3 generator reproduces the reference-generated golden curve set
  bit for bit (numpy walk and the libmrep host walk);
* the C oracle reproduces the reference's per-curve projection outputs of
  the golden set bit for bit (tests/golden/batch_mixed.npz, made by
  make_golden.py from the unmodified reference).
"""
import numpy as np
import pytest

from conftest import load_golden


def golden_set():
    g = load_golden("batch_mixed.npz")
    return g


@pytest.mark.parametrize("native", [False, True])
def test_generator_reproduces_reference_curves(native):
    from paper_2504_11498_b200.fixtures import mixed_curve_batch
    g = golden_set()
    curves = mixed_curve_batch(len(g["degree"]), max_control=int(g["max_control"]), native=native)
    co = 0
    for i, c in enumerate(curves):
        assert c.degree == g["degree"][i]
        n = c.control_points.shape[0]
        assert n == g["n_control"][i]
        assert np.array_equal(np.array(c.knots.knots),
                              g["knots"][g["knot_ofs"][i]: g["knot_ofs"][i + 1]])
        assert np.array_equal(c.control_points, g["ctrl"][co: co + n])
        co += n


def test_generator_cfg3_shape():
    from paper_2504_11498_b200.fixtures import mixed_curve_batch
    curves = mixed_curve_batch(400)
    deg = np.array([c.degree for c in curves])
    n = np.array([c.control_points.shape[0] for c in curves])
    assert deg.min() == 3 and deg.max() == 9
    assert n.min() >= 8 and n.max() <= 2048
    assert np.all(n >= deg + 1)


def test_oracle_matches_reference_per_curve(oracle_lib):
    g = golden_set()
    ofs = g["seg_ofs"]
    for c in range(len(ofs) - 1):
        a, b = ofs[c], ofs[c + 1]
        pts, ta, tb = g["seg_pts"][a:b], g["seg_ta"][a:b], g["seg_tb"][a:b]
        seam_t = np.concatenate(([ta[0]], tb))
        seam_pt = np.concatenate((pts[:1, 0], pts[:, 3]))
        m = g["curve_ids"] == c
        o = oracle_lib.project_block(pts, ta, tb, seam_t, seam_pt, g["queries"][m], workers=4)
        assert np.array_equal(o["t"], g["t"][m])
        assert np.array_equal(o["dist"], g["dist"][m])
        assert np.array_equal(o["foot"], g["foot"][m])
        assert np.array_equal(o["cand"], g["cand"][m])


def test_project_batch_validates_before_device():
    from paper_2504_11498_b200 import DomainError, PreparedCurveSet, project_batch

    class Fake(PreparedCurveSet):
        def __init__(self):
            self.curves = [None, None]
            self.d = 3

    fs = Fake()
    with pytest.raises(DomainError):
        project_batch(fs, np.zeros((3, 2)), [0, 1, 1])
    with pytest.raises(DomainError):
        project_batch(fs, np.zeros((3, 3)), [0, 1])
    with pytest.raises(DomainError):
        project_batch(fs, np.zeros((2, 3)), [0, 2])
    with pytest.raises(DomainError):
        project_batch(fs, np.zeros((2, 3)), [-1, 0])
    with pytest.raises(DomainError):
        project_batch(fs, np.zeros((2, 3)), [0, 0], max_iterations=0)
