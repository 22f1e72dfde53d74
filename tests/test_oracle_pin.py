"""Pin the CPU oracle to the reference's own outputs (tests/golden, produced
by tests/golden/make_golden.py from the unmodified reference).  Bit-exact."""
import numpy as np
import pytest

from conftest import load_golden, project_fixture_names


def test_quartic_roots_bit_exact(oracle_lib):
    g = load_golden("quartic.npz")
    r, c = oracle_lib.quartic_block(g["coeffs"])
    assert np.array_equal(c, g["counts"])
    m = np.isfinite(g["roots"])
    assert np.array_equal(r[m], g["roots"][m])


def test_newton_baseline_bit_exact(oracle_lib):
    g = load_golden("quartic.npz")
    r, c = oracle_lib.newton_quartic_block(g["coeffs"])
    assert np.array_equal(c, g["newton_counts"])
    m = np.isfinite(g["newton_roots"])
    assert np.array_equal(r[m], g["newton_roots"][m])


def test_scalar_ops_bit_exact(oracle_lib):
    o = load_golden("ops.npz")
    O = oracle_lib
    e = np.array([O.distance_poly(P, q) for P, q in zip(o["dp_P"], o["dp_q"])])
    assert np.array_equal(e, o["dp_e"])
    e2 = np.array([O.distance_poly(P, q) for P, q in zip(o["dp_P2"], o["dp_q2"])])
    assert np.array_equal(e2, o["dp_e2"])
    R = np.array([O.restrict_ordinates(b, lo, hi)
                  for b, lo, hi in zip(o["rs_b"], o["rs_lo"], o["rs_hi"])])
    assert np.array_equal(R, o["rs_out"])
    for b, f, z in zip(o["hull_b"], o["hull_found"], o["hull_z"]):
        got = O.hull_cross(b)
        assert got[0] == bool(f) and (got[1], got[2]) == tuple(z)
    for i in range(len(o["clip_b"])):
        it = int(o["clip_iters"][i])
        r, ok, used, w = O.clip_root(o["clip_b"][i], o["clip_tol"][i], it)
        assert (r, ok, used) == (o["clip_root"][i], bool(o["clip_ok"][i]), o["clip_used"][i])
        assert np.array_equal(w, o["clip_widths"][i][:it])
    ev = np.array([O.eval_ordinates(b, u) for b, u in zip(o["rs_b"], o["ev_u"])])
    assert np.array_equal(ev, o["ev_out"])
    pt = np.array([O.decasteljau_point(P, u) for P, u in zip(o["dp_P"], o["ev_u"])])
    assert np.array_equal(pt, o["pt_out"])


@pytest.mark.parametrize("name", project_fixture_names())
def test_project_block_bit_exact(oracle_lib, name):
    z = load_golden(f"project_{name}.npz")
    out = oracle_lib.project_block(z["seg_pts"], z["seg_ta"], z["seg_tb"], z["seam_t"],
                                   z["seam_pt"], z["queries"], float(z["clip_tol"]),
                                   int(z["max_iter"]), int(z["soundness"]), workers=4)
    for k in ("t", "foot", "dist", "cand", "stats", "sound"):
        assert np.array_equal(out[k], z[k]), k


def test_worker_count_invariance(oracle_lib):
    z = load_golden("project_table_n.npz")
    a = (z["seg_pts"], z["seg_ta"], z["seg_tb"], z["seam_t"], z["seam_pt"], z["queries"])
    o1 = oracle_lib.project_block(*a, workers=1)
    o7 = oracle_lib.project_block(*a, workers=7)
    for k in ("t", "foot", "dist", "cand", "seg"):
        assert np.array_equal(o1[k], o7[k])


def _golden_curves():
    g = load_golden("prep.npz")
    for ci in range(len(g["degree"])):
        d = int(g["dim"][ci])
        yield (ci, int(g["degree"][ci]), g["knots"][g["knot_ofs"][ci]: g["knot_ofs"][ci + 1]],
               g["ctrl"][g["ctrl_ofs"][ci]: g["ctrl_ofs"][ci + 1], :d], d)


def test_prep_oracle_bit_exact():
    """decompose + approximate restatement == reference on every golden curve."""
    from oracle import prep as P
    g = load_golden("prep.npz")
    bz = 0
    for ci, p, knots, ctrl, d in _golden_curves():
        segs = P.decompose(p, knots, ctrl)
        for Q, iv in segs:
            ref = g["bz_pts"][g["bz_ofs"][bz]: g["bz_ofs"][bz + 1], :d]
            assert np.array_equal(ref, Q) and tuple(g["bz_iv"][bz]) == iv
            bz += 1
        cub = P.approximate(segs, 1e-4)
        sel = np.nonzero(g["cu_curve"] == ci)[0]
        assert len(sel) == len(cub)
        for k, (Pc, iv, err) in zip(sel, cub):
            assert np.array_equal(g["cu_pts"][k][:, :d], Pc)
            assert tuple(g["cu_iv"][k]) == iv and g["cu_err"][k] == err
    assert bz == len(g["bz_iv"])


def test_prepared_tables_match_golden():
    from oracle import prep as P
    for name in ("cfg1_random", "table_n", "kink", "deg9"):
        z = load_golden(f"project_{name}.npz")
        pr = P.prepare(int(z["degree"]), z["knots"], z["ctrl"], float(z["tolerance"]))
        for k in ("seg_pts", "seg_ta", "seg_tb", "seam_t", "seam_pt"):
            assert np.array_equal(pr[k], z[k]), (name, k)


def test_fixture_generator_matches_golden_curves():
    from oracle import prep as P
    z = load_golden("project_cfg2.npz")
    p, knots, ctrl = P.clamped_uniform_curve(np.random.default_rng(0), 7, 512, 3)
    assert np.array_equal(knots, z["knots"]) and np.array_equal(ctrl, z["ctrl"])
    from paper_2504_11498_b200.fixtures import random_clamped_curve
    c = random_clamped_curve(np.random.default_rng(0), 3, 64, 3, uniform_knots=True)
    z1 = load_golden("project_cfg1_random.npz")
    assert np.array_equal(c.knots.knots, z1["knots"])
    assert np.array_equal(c.control_points, z1["ctrl"])
