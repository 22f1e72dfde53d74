"""Per-op device kernels vs the reference's golden vectors.

Bars: bit-exact for the pure-arithmetic ops (distance poly, restriction,
hull, clipping, evaluation) -- FMA contraction is off and the operation
order is the reference's.  The quartic solver calls acos/cos/cbrt, where
CUDA's libm differs from glibc by ulps; root COUNTS must match exactly and
roots within 1e-8 (the reference's own bisection-oracle bar, test_distance.py:78-86;
near-double roots amplify an ulp in the resolvent to ~1e-9).
"""
import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def test_quartic_roots(gpu):
    from paper_2504_11498_b200 import _device as D
    g = load_golden("quartic.npz")
    r, c = D.quartic_roots(g["coeffs"])
    assert np.array_equal(c, g["counts"])
    m = np.isfinite(g["roots"])
    assert np.abs(r[m] - g["roots"][m]).max() <= 1e-8
    assert np.mean(r[m] == g["roots"][m]) >= 0.9


def test_newton_quartic_baseline(gpu):
    from paper_2504_11498_b200 import _device as D
    g = load_golden("quartic.npz")
    r, c = D.newton_quartic_roots(g["coeffs"])
    assert np.array_equal(c, g["newton_counts"])
    m = np.isfinite(g["newton_roots"])
    assert np.array_equal(r[m], g["newton_roots"][m])


def test_distance_poly_bit_exact(gpu):
    from paper_2504_11498_b200 import _device as D
    o = load_golden("ops.npz")
    assert np.array_equal(D.distance_poly(o["dp_P"], o["dp_q"]), o["dp_e"])
    assert np.array_equal(D.distance_poly(o["dp_P2"], o["dp_q2"]), o["dp_e2"])


def test_restrict_hull_eval_bit_exact(gpu):
    from paper_2504_11498_b200 import _device as D
    o = load_golden("ops.npz")
    assert np.array_equal(D.restrict_ordinates(o["rs_b"], o["rs_lo"], o["rs_hi"]), o["rs_out"])
    f, z = D.hull_cross(o["hull_b"])
    assert np.array_equal(f, o["hull_found"].astype(bool))
    assert np.array_equal(z, o["hull_z"])
    assert np.array_equal(D.eval_ordinates(o["rs_b"], o["ev_u"]), o["ev_out"])
    assert np.array_equal(D.cubic_points(o["dp_P"], o["ev_u"]), o["pt_out"])


@pytest.mark.parametrize("iters", [3, 8])
@pytest.mark.parametrize("tol", [1e-9, 1e-6])
def test_clip_root_bit_exact(gpu, iters, tol):
    from paper_2504_11498_b200 import _device as D
    o = load_golden("ops.npz")
    sel = (o["clip_iters"] == iters) & (o["clip_tol"] == tol)
    root, ok, used, w = D.clip_root(o["clip_b"][sel], tol, iters)
    assert np.array_equal(root, o["clip_root"][sel])
    assert np.array_equal(ok, o["clip_ok"][sel].astype(bool))
    assert np.array_equal(used, o["clip_used"][sel])
    assert np.array_equal(w, o["clip_widths"][sel][:, :iters])


def test_rebase_matches_T5(gpu):
    from paper_2504_11498_b200 import _device as D
    o = load_golden("ops.npz")
    e = o["dp_e"]
    ref = e @ o["T5"].T
    assert np.abs(D.rebase(e) - ref).max() <= 1e-13 * max(1.0, np.abs(e).max())


def test_oracle_agrees_on_random_quartics(gpu, oracle_lib):
    """Fresh random inputs (not in the goldens) vs the pinned C oracle."""
    from paper_2504_11498_b200 import _device as D
    c = np.random.default_rng(99).uniform(-1, 1, (20000, 5))
    r, cnt = D.quartic_roots(c)
    ro, co = oracle_lib.quartic_block(c)
    assert np.mean(cnt == co) >= 0.9995
    same = cnt == co
    m = np.isfinite(ro[same])
    assert np.abs(r[same][m] - ro[same][m]).max() <= 1e-8
