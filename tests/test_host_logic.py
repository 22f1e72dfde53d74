"""Host-side API logic (no device): validation, errors, bookkeeping ops."""
import numpy as np
import pytest

from conftest import load_golden
from paper_2504_11498_b200 import (
    BSplineCurve,
    CountMismatch,
    DegreeOutOfRange,
    DomainError,
    NonMonotoneKnots,
    NotClamped,
    Poly,
    global_to_local,
    local_to_global,
    plan_work,
    reduce_min,
    validate_curve,
)
from paper_2504_11498_b200.basis import (
    bernstein_matrix,
    bernstein_matrix_inverse,
    gram_matrix,
    power_to_bernstein_matrix,
    subdivision_matrices,
)


class TestValidate:
    def test_ok(self):
        c = BSplineCurve(3, [0, 0, 0, 0, 1, 1, 1, 1], np.zeros((4, 2)))
        assert validate_curve(c) is c

    def test_degree(self):
        with pytest.raises(DegreeOutOfRange):
            validate_curve(BSplineCurve(32, [0] * 33 + [1] * 33, np.zeros((33, 2))))

    def test_nonmonotone(self):
        with pytest.raises(NonMonotoneKnots):
            validate_curve(BSplineCurve(1, [0, 0, 0.6, 0.4, 1, 1], np.zeros((4, 2))))

    def test_not_clamped(self):
        with pytest.raises(NotClamped):
            validate_curve(BSplineCurve(2, [0, 0, 0.1, 0.5, 1, 1, 1], np.zeros((4, 2))))

    def test_count(self):
        with pytest.raises(CountMismatch):
            validate_curve(BSplineCurve(3, [0, 0, 0, 0, 1, 1, 1, 1], np.zeros((5, 2))))

    def test_multiplicity(self):
        with pytest.raises(NonMonotoneKnots):
            validate_curve(BSplineCurve(2, [0, 0, 0, 0.5, 0.5, 0.5, 0.5, 1, 1, 1],
                                        np.zeros((7, 2))))

    def test_dimension(self):
        with pytest.raises(DomainError):
            validate_curve(BSplineCurve(1, [0, 0, 1, 1], np.zeros((2, 4))))


def test_param_maps_roundtrip():
    iv = (2.0, 12.0)
    for u in np.linspace(0, 1, 17):
        assert abs(global_to_local(iv, local_to_global(iv, u)) - u) <= 1e-14
    with pytest.raises(DomainError):
        local_to_global(iv, 1.5)


def test_poly():
    p = Poly([1.0, -2.0, 3.0])
    assert p(2.0) == 9.0
    assert np.array_equal(p.derivative().coeffs, [-2.0, 6.0])
    assert Poly([1.0, 0.0, 1e-14]).effective_degree() == 0


def test_plan_work():
    assert plan_work(100, 7).units_per_worker == 15
    assert plan_work(3, 8).units_per_worker == 1
    with pytest.raises(DomainError):
        plan_work(10, 0)


def test_reduce_min_tie_band():
    cands = [(0.456, np.zeros(2), 1e-9 + 5e-13), (0.123, np.zeros(2), 1e-9),
             (0.9, np.zeros(2), 5.0)]
    r = reduce_min(np.zeros(2), cands)
    assert r.t_star == 0.123 and r.candidates_examined == 3


def test_constant_matrices_match_reference_goldens():
    o = load_golden("ops.npz")
    assert np.array_equal(power_to_bernstein_matrix(5), o["T5"])
    assert np.array_equal(bernstein_matrix(3), o["B3"])
    for p in (3, 5, 9):
        assert np.abs(power_to_bernstein_matrix(p) @ bernstein_matrix(p)
                      - np.eye(p + 1)).max() < 1e-12
        assert np.abs(bernstein_matrix_inverse(p) - power_to_bernstein_matrix(p)).max() < 1e-9
    assert abs(gram_matrix(3, 3).sum() - 1.0) < 1e-15
    SL, SR = subdivision_matrices(0.3)
    assert np.allclose(SL.sum(1), 1.0) and np.allclose(SR.sum(1), 1.0)


def test_table_layout_levels():
    """8-ary box hierarchy sizes used by the device table."""
    from paper_2504_11498_b200 import _lib
    lib = _lib.load_library()
    for S in (1, 7, 8, 9, 64, 65, 100_000):
        cnt, lv, boxes = S, 0, 0
        while True:
            boxes += cnt
            if lv >= 1 and cnt <= 1:
                break
            cnt = (cnt + 7) // 8
            lv += 1
        # 6 doubles per box + its float copy (6 floats), the compact seam
        # block, then the tensor-core B fragments (32-B aligned, 2 of slack)
        n = 64 + 32 * S + 9 * boxes + 3 * (S + 1)
        assert lib.mrep_table_bytes(S) == (((n + 3) // 4) * 4 + 32 * (S + 2)) * 8


def test_nearest_set_locate():
    """Global winning index -> (curve, local cubic); the separator before a
    curve maps to that curve's cubic 0 (a seam candidate at its start)."""
    from paper_2504_11498_b200.nearest import PreparedNearestSet
    ns = object.__new__(PreparedNearestSet)
    ns.counts = np.array([3, 1, 4])
    ns.starts = np.array([0, 4, 6])  # cubics 0-2, sep 3, cubic 4, sep 5, cubics 6-9
    cid, local = ns.locate([0, 2, 3, 4, 5, 6, 9])
    assert cid.tolist() == [0, 0, 1, 1, 2, 2, 2]
    assert local.tolist() == [0, 2, 0, 0, 0, 0, 3]
