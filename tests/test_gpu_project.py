"""Batch projection kernel (dense = reference semantics, screened = BVH) vs
the reference's golden outputs and the pinned C oracle.

Bars (north star): segment index exact except ties the oracle itself
detects (another segment within dmin + 2e-12); distance within 1e-9 relative
(absolute floor 1e-12 for on-curve queries, whose distance is ~0); parameter
within 1e-6.  Dense mode must also reproduce the reference's candidate count
and all six stats columns exactly.
"""
import numpy as np
import pytest

from conftest import assert_parity, load_golden, project_fixture_names

pytestmark = pytest.mark.gpu


def _args(z):
    return (z["seg_pts"], z["seg_ta"], z["seg_tb"], z["seam_t"], z["seam_pt"])


def assert_close(t, dist, t_ref, d_ref):
    assert np.all(np.abs(t - t_ref) <= 1e-6), np.abs(t - t_ref).max()
    tol = np.maximum(1e-9 * d_ref, 1e-12)
    assert np.all(np.abs(dist - d_ref) <= tol), np.abs(dist - d_ref).max()


@pytest.mark.parametrize("name", project_fixture_names())
def test_dense_matches_reference(gpu, name):
    from paper_2504_11498_b200 import _device as D
    z = load_golden(f"project_{name}.npz")
    t, foot, dist, cand, stats, sound = D.project_block(
        *_args(z), z["queries"], float(z["clip_tol"]), int(z["max_iter"]), int(z["soundness"]))
    assert_close(t, dist, z["t"], z["dist"])
    assert np.abs(foot - z["foot"]).max() <= 1e-6
    assert np.array_equal(cand, z["cand"])
    assert np.array_equal(stats, z["stats"])
    if int(z["soundness"]) > 0:
        fin = np.isfinite(z["sound"])
        assert np.array_equal(np.isfinite(sound), fin)
        assert np.abs(sound[fin] - z["sound"][fin]).max() <= 1e-9


@pytest.mark.parametrize("name", project_fixture_names())
def test_wavefront_fused_unsorted_agree(gpu, name):
    """The three screened schedules (wavefront, fused warp kernel, input
    order) produce bit-identical winners."""
    from paper_2504_11498_b200 import _device as D, _lib as L
    z = load_golden(f"project_{name}.npz")
    tab = D.DeviceTable(*_args(z))
    a = tab.project(z["queries"])
    b = tab.project(z["queries"], extra_flags=L.MREP_FUSED)
    c = tab.project(z["queries"], extra_flags=L.MREP_NO_SORT | L.MREP_FUSED)
    d = tab.project(z["queries"], extra_flags=L.MREP_PACKET)
    e = tab.project(z["queries"], extra_flags=L.MREP_PER_LANE)
    f = tab.project(z["queries"], extra_flags=L.MREP_GROUP)
    tab.build_cells()
    g = tab.project(z["queries"], extra_flags=L.MREP_CELLS)
    for k in (0, 1, 2, 4):
        for other in (b, c, d, e, f, g):
            assert np.array_equal(a[k].cpu().numpy(), other[k].cpu().numpy()), k


@pytest.mark.parametrize("name", project_fixture_names())
def test_screened_equals_dense(gpu, name):
    """The BVH cull never changes the winner: bitwise equal to brute force."""
    from paper_2504_11498_b200 import _device as D
    z = load_golden(f"project_{name}.npz")
    tab = D.DeviceTable(*_args(z))
    dense = tab.project(z["queries"], screen=False)
    scr = tab.project(z["queries"], screen=True)
    for a, b in zip(dense[:5], scr[:5]):
        if a is not None:
            pass
    for k in (0, 1, 2, 4):  # t, foot, dist, seg
        assert np.array_equal(dense[k].cpu().numpy(), scr[k].cpu().numpy()), k
    assert_close(scr[0].cpu().numpy(), scr[2].cpu().numpy(), z["t"], z["dist"])


def test_segment_ids_match_oracle(gpu, oracle_lib):
    """Winning cubic index (the north star's 'segment id') vs the oracle."""
    from paper_2504_11498_b200 import _device as D
    for name in project_fixture_names():
        z = load_golden(f"project_{name}.npz")
        o = oracle_lib.project_block(*_args(z), z["queries"], workers=8)
        tab = D.DeviceTable(*_args(z))
        for screen in (True, False):
            r = [x.cpu().numpy() for x in tab.project(z["queries"], screen=screen)[:5]]
            assert_parity(r[0], r[2], r[4], o)


def test_cfg2_random_vs_oracle(gpu, oracle_lib):
    """Fresh cfg2 queries (20k, S = 510) vs the C oracle on all host cores."""
    from paper_2504_11498_b200 import _device as D
    import os
    z = load_golden("project_cfg2.npz")
    q = np.random.default_rng(123).uniform(0, 1, (20000, 3))
    o = oracle_lib.project_block(*_args(z), q, workers=os.cpu_count() or 1)
    tab = D.DeviceTable(*_args(z))
    t, foot, dist, cand, seg, _, _ = [x.cpu().numpy() if x is not None else None
                                      for x in tab.project(q)]
    assert_parity(t, dist, seg, o)
    assert np.mean(t == o["t"]) >= 0.99


def test_full_size_properties(gpu):
    """10^6 queries at cfg2 size: determinism, seam upper bound, dense agreement
    on a subsample, foot point lies on the winning cubic."""
    import torch
    from paper_2504_11498_b200 import _device as D
    z = load_golden("project_cfg2.npz")
    tab = D.DeviceTable(*_args(z))
    g = torch.Generator(device="cuda").manual_seed(7)
    q = torch.rand((1_000_000, 3), dtype=torch.float64, device="cuda", generator=g)
    a = tab.project(q)
    b = tab.project(q)
    for k in (0, 1, 2, 4):
        assert torch.equal(a[k], b[k])
    seam = torch.as_tensor(z["seam_pt"], device="cuda")
    sub = q[::997]
    dseam = ((sub[:, None, :] - seam[None]) ** 2).sum(-1).sqrt().min(dim=1).values
    assert bool((a[2][::997] <= dseam + 1e-15).all())
    dn = tab.project(sub, screen=False)
    for k in (0, 1, 2, 4):
        assert torch.equal(dn[k], a[k][::997])
    # foot consistency: distance == |q - foot|
    assert float((a[2] - (q - a[1]).norm(dim=1)).abs().max()) <= 1e-12


def test_tie_band_overflow_second_pass(gpu, oracle_lib):
    """Many candidates inside the 1e-12 band (query at the centre of a
    polygon inscribed in a circle): the exact second pass must give the
    reference's choice (smallest t among the band)."""
    from paper_2504_11498_b200 import _device as D, _lib as L
    import torch
    k = 24
    ang = np.linspace(0, 2 * np.pi, k, endpoint=False)
    # cubic segments that are straight chords between points on the circle
    P0 = np.stack([np.cos(ang), np.sin(ang)], 1)
    P3 = np.roll(P0, -1, axis=0)
    seg_pts = np.stack([P0, P0 + (P3 - P0) / 3, P0 + 2 * (P3 - P0) / 3, P3], 1)
    ta = np.arange(k) / k
    tb = np.arange(1, k + 1) / k
    seam_t = np.concatenate(([0.0], tb))
    seam_pt = np.concatenate((seg_pts[:1, 0], seg_pts[:, 3]))
    q = np.array([[0.0, 0.0], [1e-3, -2e-3], [0.5, 0.1]])
    o = oracle_lib.project_block(seg_pts, ta, tb, seam_t, seam_pt, q)
    tab = D.DeviceTable(seg_pts, ta, tb, seam_t, seam_pt)
    cnt = torch.zeros(L.NUM_COUNTERS, dtype=torch.int64, device="cuda")
    for screen in (False, True):
        t, foot, dist, cand, seg, _, _ = tab.project(q, screen=screen, counters=cnt)
        assert np.array_equal(t.cpu().numpy(), o["t"])
        assert np.array_equal(dist.cpu().numpy(), o["dist"])
        assert np.array_equal(seg.cpu().numpy(), o["seg"])
    assert int(cnt[L.CNT_PASS2]) >= 1


def test_edge_queries(gpu, oracle_lib):
    """Far-away, on-seam, on-endpoint queries and a single query."""
    from paper_2504_11498_b200 import _device as D
    z = load_golden("project_table_n.npz")
    q = np.concatenate([z["seam_pt"], np.array([[1e6, -1e6, 3e5], [0.5, 0.5, 0.5]]),
                        z["seg_pts"][:, 1]])
    o = oracle_lib.project_block(*_args(z), q)
    tab = D.DeviceTable(*_args(z))
    for screen in (False, True):
        t, foot, dist, cand, seg, _, _ = [x.cpu().numpy() if x is not None else None
                                          for x in tab.project(q, screen=screen)]
        assert_close(t, dist, o["t"], o["dist"])
    one = tab.project(q[:1])
    assert one[0].shape == (1,)
    assert np.all(np.isfinite(tab.project(q)[0].cpu().numpy()))


def _star_polyline(k=12, dim=2):
    """Degree-1 closed star: inner vertices exactly at distance 5 from the
    origin (integer Pythagorean points), outer ones at radius 10 between
    them -- every inner vertex (a seam) is an exact tie for the nearest
    point of the origin, more than the 4-slot tie band holds."""
    from paper_2504_11498_b200 import BSplineCurve
    inner = [(5, 0), (4, 3), (3, 4), (0, 5), (-3, 4), (-4, 3), (-5, 0), (-4, -3), (-3, -4),
             (0, -5), (3, -4), (4, -3)][:k]
    pts = []
    for i, (x, y) in enumerate(inner):
        pts.append((float(x), float(y)))
        a0 = np.arctan2(y, x)
        x1, y1 = inner[(i + 1) % len(inner)]
        a1 = np.arctan2(y1, x1)
        am = a0 + 0.5 * ((a1 - a0 + np.pi) % (2 * np.pi) - np.pi)
        pts.append((10.0 * np.cos(am), 10.0 * np.sin(am)))
    pts.append(pts[0])
    P = np.array(pts)
    if dim == 3:
        P = np.concatenate([P, np.zeros((len(P), 1))], axis=1)
    n = len(P)
    knots = np.concatenate(([0.0], np.linspace(0.0, 1.0, n), [1.0]))
    return BSplineCurve(1, knots, P)


@pytest.mark.parametrize("dim", [2, 3])
def test_exact_seam_ties_overflow_band(gpu, oracle_lib, dim):
    """Twelve seams tie exactly for the origin: the screened kernel's tie band
    overflows and the exact second pass / fallback must pick the reference's
    winner (smallest t among the tied seams)."""
    from paper_2504_11498_b200 import _lib as L, prepare_curve
    from paper_2504_11498_b200 import _device as D
    curve = _star_polyline(12, dim)
    prep = prepare_curve(curve, 1e-4)
    q = np.zeros((64, dim))
    q[1:] = np.random.default_rng(0).uniform(-12, 12, (63, dim))
    o = oracle_lib.project_block(prep.seg_pts, prep.seg_ta, prep.seg_tb, prep.seam_t,
                                 prep.seam_pt, q)
    assert o["dist"][0] == 5.0 and o["t"][0] == 0.0
    tab = prep.table
    cnt = np.zeros(L.NUM_COUNTERS, dtype=np.uint64)
    outs = [tab.project(q, screen=s, extra_flags=f)
            for s, f in ((False, 0), (True, 0), (True, L.MREP_GROUP), (True, L.MREP_PER_LANE),
                         (True, L.MREP_FUSED))]
    for out in outs:
        t, foot, dist = out[0].cpu().numpy(), out[1].cpu().numpy(), out[2].cpu().numpy()
        assert np.array_equal(t, o["t"]) or np.abs(t - o["t"]).max() <= 1e-12
        assert np.abs(dist - o["dist"]).max() <= 1e-12
        assert t[0] == 0.0 and dist[0] == 5.0
    for a, b in zip(outs[0][:3], outs[1][:3]):
        assert np.array_equal(a.cpu().numpy(), b.cpu().numpy())


@pytest.mark.parametrize("scale", [1e-6, 1e6])
def test_scaled_geometry(gpu, oracle_lib, scale):
    """The cfg1 curve and queries scaled by 1e-6 / 1e6: screening margins are
    relative, results still match the reference kernel's."""
    from paper_2504_11498_b200 import BSplineCurve, prepare_curve, project_prepared
    z = load_golden("project_cfg1_random.npz")
    curve = BSplineCurve(int(z["degree"]), z["knots"], z["ctrl"] * scale)
    prep = prepare_curve(curve, 1e-4 * scale)
    q = z["queries"] * scale
    t, foot, dist, cand = project_prepared(prep, q)
    o = oracle_lib.project_block(prep.seg_pts, prep.seg_ta, prep.seg_tb, prep.seam_t,
                                 prep.seam_pt, q, workers=8)
    assert np.all(np.abs(t - o["t"]) <= 1e-6)
    assert np.all(np.abs(dist - o["dist"]) <= np.maximum(1e-9 * o["dist"], 1e-12 * scale))


def test_degenerate_and_far_queries(gpu, oracle_lib):
    """A curve with coincident control points (zero-length cubic pieces) and
    queries far outside the table box."""
    from paper_2504_11498_b200 import BSplineCurve, prepare_curve, project_prepared
    P = np.array([[0, 0, 0], [0, 0, 0], [0, 0, 0], [1, 1, 0], [1, 1, 0], [2, 0, 1], [2, 0, 1]],
                 dtype=np.float64)
    knots = np.concatenate(([0.0] * 4, [0.25, 0.5, 0.75], [1.0] * 4))
    curve = BSplineCurve(3, knots, P)
    prep = prepare_curve(curve, 1e-4)
    rng = np.random.default_rng(3)
    q = np.concatenate([rng.uniform(-1, 3, (500, 3)), rng.uniform(-1e7, 1e7, (20, 3)),
                        P[[0, -1]]])
    t, foot, dist, cand = project_prepared(prep, q)
    o = oracle_lib.project_block(prep.seg_pts, prep.seg_ta, prep.seg_tb, prep.seam_t,
                                 prep.seam_pt, q, workers=8)
    assert np.all(np.abs(t - o["t"]) <= 1e-6)
    assert np.all(np.abs(dist - o["dist"]) <= np.maximum(1e-9 * o["dist"], 1e-12))
    assert dist[-2:].max() <= 1e-12  # the clamped ends lie on the curve


@pytest.mark.parametrize("grid", [8, 64])
def test_cell_index_bitwise_equal_to_tree_walk(gpu, grid):
    """cfg2 curve, 2e5 queries (some outside the grid): the cell-index
    traversal gives the tree walk's results bit for bit."""
    from paper_2504_11498_b200 import _lib as L
    from paper_2504_11498_b200 import _device as D
    z = load_golden("project_cfg2.npz")
    tab = D.DeviceTable(z["seg_pts"], z["seg_ta"], z["seg_tb"], z["seam_t"], z["seam_pt"])
    rng = np.random.default_rng(8)
    q = np.concatenate([rng.uniform(0, 1, (200000, 3)), rng.uniform(-3, 4, (2000, 3))])
    a = tab.project(q, extra_flags=L.MREP_PACKET)
    tab.build_cells(grid)
    b = tab.project(q, extra_flags=L.MREP_CELLS)
    for k in (0, 1, 2, 4):
        assert np.array_equal(a[k].cpu().numpy(), b[k].cpu().numpy()), k


def test_cell_index_large_table_bvh_build(gpu):
    """A 2e4-cubic curve (cell lists built by walking the hierarchy, not by
    brute force): cell traversal == tree walk bit for bit."""
    from paper_2504_11498_b200 import BSplineCurve, _lib as L, prepare_curve
    from paper_2504_11498_b200.fixtures import random_clamped_curve
    cv = random_clamped_curve(np.random.default_rng(17), 3, 20003, 3, uniform_knots=True,
                              native=True)
    prep = prepare_curve(cv, 1e-4)
    assert prep.num_segments == 20000
    tab = prep.table
    q = np.random.default_rng(18).uniform(-0.1, 1.1, (150000, 3))
    a = tab.project(q, extra_flags=L.MREP_PACKET)
    tab.build_cells(24)
    b = tab.project(q, extra_flags=L.MREP_CELLS)
    for k in (0, 1, 2, 4):
        assert np.array_equal(a[k].cpu().numpy(), b[k].cpu().numpy()), k


def test_cand_deterministic_with_bucket_order(gpu):
    """Cell / per-lane walks take the bucket-sorted order (queries of one
    bucket in no fixed order); every output, `cand` included, is a function of
    the query alone: repeated calls and a sub-batch agree bit for bit."""
    from paper_2504_11498_b200 import _lib as L
    from paper_2504_11498_b200 import _device as D
    z = load_golden("project_cfg2.npz")
    tab = D.DeviceTable(z["seg_pts"], z["seg_ta"], z["seg_tb"], z["seam_t"], z["seam_pt"])
    tab.build_cells(32)
    q = np.random.default_rng(21).uniform(-0.2, 1.2, (100000, 3))
    for flags in (L.MREP_CELLS, L.MREP_PER_LANE, L.MREP_GROUP):
        a = [x.cpu().numpy() for x in tab.project(q, extra_flags=flags)[:5]]
        b = [x.cpu().numpy() for x in tab.project(q, extra_flags=flags)[:5]]
        c = [x.cpu().numpy() for x in tab.project(q[:7777], extra_flags=flags)[:5]]
        for x, y, zz in zip(a, b, c):
            assert np.array_equal(x, y)
            assert np.array_equal(x[:7777], zz)


@pytest.mark.parametrize("flags", ["default", "packet", "lane"])
def test_sorted_and_unsorted_agree(gpu, flags):
    """Batches of >= 2^16 queries are bucket- or radix-sorted, smaller ones
    are not: the outputs never depend on the order (bit for bit)."""
    from paper_2504_11498_b200 import _lib as L
    from paper_2504_11498_b200 import _device as D
    z = load_golden("project_cfg2.npz")
    tab = D.DeviceTable(z["seg_pts"], z["seg_ta"], z["seg_tb"], z["seam_t"], z["seam_pt"])
    q = np.random.default_rng(31).uniform(-0.1, 1.1, (70000, 3))
    f = {"default": 0, "packet": L.MREP_PACKET, "lane": L.MREP_PER_LANE}[flags]
    a = [x.cpu().numpy() for x in tab.project(q, extra_flags=f)[:5]]
    b = [x.cpu().numpy() for x in tab.project(q, extra_flags=f | L.MREP_NO_SORT)[:5]]
    for k in (0, 1, 2, 4):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("name", project_fixture_names())
def test_exact_cand_matches_reference(gpu, name):
    """MREP_CAND_EXACT (the Python default): the tensor-core sign screen plus
    the exact solve of undecided pairs reproduces the reference's candidate
    count bit for bit, in every traversal mode and through the host call."""
    from paper_2504_11498_b200 import _device as D, _lib as L
    z = load_golden(f"project_{name}.npz")
    tab = D.DeviceTable(*_args(z))
    for fl in (0, L.MREP_PACKET, L.MREP_GROUP):
        r = tab.project(z["queries"], extra_flags=L.MREP_CAND_EXACT | fl)
        assert np.array_equal(r[3].cpu().numpy(), z["cand"]), fl
    h = tab.project_host(z["queries"], extra_flags=L.MREP_CAND_EXACT)
    assert np.array_equal(h[3], z["cand"])


def test_exact_cand_cfg2_and_extremes_vs_oracle(gpu, oracle_lib):
    """cfg2's curve (510 cubics) with random, on-curve, seam, far and
    tiny-scale queries: default project_prepared cand == the C oracle's."""
    from paper_2504_11498_b200 import BSplineCurve, prepare_curve, project_prepared
    from paper_2504_11498_b200.fixtures import random_clamped_curve
    cv = random_clamped_curve(np.random.default_rng(0), 7, 512, 3, uniform_knots=True)
    rng = np.random.default_rng(5)
    for scale in (1.0, 1e-3, 1e3):
        c2 = BSplineCurve(cv.degree, np.array(cv.knots.knots), np.array(cv.control_points) * scale)
        prep = prepare_curve(c2, 1e-4 * scale)
        q = np.concatenate([
            rng.uniform(0, scale, (3000, 3)),                  # random
            prep.seam_pt[::7],                                  # exactly on seams
            prep.seg_pts[::5, 1],                               # control points
            rng.normal(0, 1e3 * scale, (200, 3)),               # far away
        ])
        t, foot, dist, cand = project_prepared(prep, q)
        o = oracle_lib.project_block(prep.seg_pts, prep.seg_ta, prep.seg_tb, prep.seam_t,
                                     prep.seam_pt, q, workers=8)
        assert np.array_equal(cand, o["cand"]), (scale, np.nonzero(cand != o["cand"])[0][:10])
        ts, _, ds, cs = project_prepared(prep, q, cand="screened")
        assert np.array_equal(ts, t) and np.array_equal(ds, dist)
        assert np.all(cs <= cand)


@pytest.mark.parametrize("grid", [8, 32])
def test_cand_cell_index_exact(gpu, oracle_lib, grid):
    """The cand cell index (mrep_cand_cells_build) changes no count: per cell
    the certified cubics (zero or exactly one survivor for every query of the
    cell) are skipped and the rest tested per query.  Checked against the
    full tensor-core pass and the C oracle, with queries outside the grid,
    on seams and control points, at three coordinate scales; sorted (>= 2^16
    queries) and unsorted batches; the host call."""
    from paper_2504_11498_b200 import BSplineCurve, prepare_curve, _lib as L
    from paper_2504_11498_b200.fixtures import random_clamped_curve
    cv = random_clamped_curve(np.random.default_rng(0), 7, 512, 3, uniform_knots=True)
    rng = np.random.default_rng(6)
    for scale in (1.0, 1e-3, 1e3):
        c2 = BSplineCurve(cv.degree, np.array(cv.knots.knots), np.array(cv.control_points) * scale)
        prep = prepare_curve(c2, 1e-4 * scale)
        tab = prep.table
        q = np.concatenate([
            rng.uniform(0, scale, (70000, 3)),                  # random (sorted batch)
            rng.uniform(-0.5 * scale, 1.5 * scale, (3000, 3)),  # many outside the grid
            prep.seam_pt[::3],                                  # exactly on seams
            prep.seg_pts[::2, 1],                               # control points
        ])
        tab.cand_tried = True  # no lazy index: the full pass
        full = tab.project(q, extra_flags=L.MREP_CAND_EXACT)[3].cpu().numpy()
        tab.build_cand_cells(grid)
        assert tab.cand_cells is not None
        fl = L.MREP_CAND_EXACT | L.MREP_CAND_CELLS
        idx = tab.project(q, extra_flags=fl)[3].cpu().numpy()
        assert np.array_equal(idx, full), (scale, np.nonzero(idx != full)[0][:10])
        small = tab.project(q[-4000:], extra_flags=fl)[3].cpu().numpy()  # unsorted path
        assert np.array_equal(small, full[-4000:])
        h = tab.project_host(q, extra_flags=fl)
        assert np.array_equal(h[3], full)
        sub = np.concatenate([np.arange(0, 70000, 61), np.arange(70000, len(q))])
        o = oracle_lib.project_block(prep.seg_pts, prep.seg_ta, prep.seg_tb, prep.seam_t,
                                     prep.seam_pt, q[sub], workers=8)
        assert np.array_equal(idx[sub], o["cand"])


def test_cand_cell_index_2d(gpu, oracle_lib):
    from paper_2504_11498_b200 import BSplineCurve, prepare_curve, _lib as L
    from paper_2504_11498_b200.fixtures import random_clamped_curve
    cv = random_clamped_curve(np.random.default_rng(3), 5, 200, 2, uniform_knots=True)
    prep = prepare_curve(cv, 1e-4)
    tab = prep.table
    tab.cand_tried = True
    q = np.random.default_rng(4).uniform(-0.2, 1.2, (20000, 2))
    full = tab.project(q, extra_flags=L.MREP_CAND_EXACT)[3].cpu().numpy()
    tab.build_cand_cells(64)
    idx = tab.project(q, extra_flags=L.MREP_CAND_EXACT | L.MREP_CAND_CELLS)[3].cpu().numpy()
    assert np.array_equal(idx, full)
    o = oracle_lib.project_block(prep.seg_pts, prep.seg_ta, prep.seg_tb, prep.seam_t,
                                 prep.seam_pt, q[::10], workers=8)
    assert np.array_equal(idx[::10], o["cand"])


def test_cand_cell_index_list_overflow_redo(gpu):
    """Undecided pairs that overflow the global list (forced tiny with
    MREP_CAND_GCAP) send their rows to the whole-row recount: same counts."""
    import subprocess
    import sys
    code = r"""
import numpy as np, sys
sys.path.insert(0, '.')
from paper_2504_11498_b200 import prepare_curve, _lib as L
from paper_2504_11498_b200.fixtures import random_clamped_curve
cv = random_clamped_curve(np.random.default_rng(0), 7, 300, 3, uniform_knots=True)
tab = prepare_curve(cv, 1e-4).table
tab.cand_tried = True
q = np.random.default_rng(8).uniform(-0.2, 1.2, (70000, 3))
full = tab.project(q, extra_flags=L.MREP_CAND_EXACT)[3].cpu().numpy()
tab.build_cand_cells(32)
idx = tab.project(q, extra_flags=L.MREP_CAND_EXACT | L.MREP_CAND_CELLS)[3].cpu().numpy()
assert np.array_equal(idx, full), np.nonzero(idx != full)[0][:10]
print("ok")
"""
    import os
    env = dict(os.environ, MREP_CAND_GCAP="5000")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_dmma_cell_screen_bitwise_equal(gpu):
    """MREP_TRAV_DMMA (tensor-core Bernstein screen of the cell lists, an A/B
    variant) returns the default pipeline's t / foot / distance / segment
    bit for bit, including queries outside the cell grid."""
    import os
    import subprocess
    import sys
    code = r"""
import numpy as np, sys, torch
sys.path.insert(0, '.')
from paper_2504_11498_b200 import prepare_curve
from paper_2504_11498_b200.fixtures import random_clamped_curve
cv = random_clamped_curve(np.random.default_rng(0), 7, 400, 3, uniform_knots=True)
tab = prepare_curve(cv, 1e-4).table
tab.CELL_MIN_QUERIES = 0
q = np.random.default_rng(9).uniform(-0.3, 1.3, (90000, 3))
r = tab.project(q)
np.savez(sys.argv[1], t=r[0].cpu().numpy(), f=r[1].cpu().numpy(), d=r[2].cpu().numpy(),
         s=r[4].cpu().numpy())
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for k, env in enumerate((dict(os.environ), dict(os.environ, MREP_TRAV_DMMA="1"))):
        path = os.path.join(root, "build", f"dmma_{k}.npz")
        r = subprocess.run([sys.executable, "-c", code, path], env=env, cwd=root,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
    for key in ("t", "f", "d", "s"):
        assert np.array_equal(outs[0][key], outs[1][key], equal_nan=True), key


def test_fallback_queries_in_sorted_batches(gpu, oracle_lib):
    """Batches of >= 2^16 queries take the sorted path whose outputs go
    through staging records + the unpermute pass; queries finished by the
    exact fallback (tie-band overflow at the star's centre) must keep the
    fallback's outputs, every other query the staged ones."""
    from paper_2504_11498_b200 import _lib as L, prepare_curve
    curve = _star_polyline(12, 3)
    prep = prepare_curve(curve, 1e-4)
    rng = np.random.default_rng(12)
    q = rng.uniform(-12, 12, (70000, 3))
    q[::997] = 0.0  # the tie point, scattered through the caller order
    tab = prep.table
    cnt = np.zeros(L.NUM_COUNTERS, dtype=np.uint64)
    import torch
    ct = torch.from_numpy(cnt.astype(np.int64)).cuda()
    t, foot, dist, cand, seg, _, _ = tab.project(q, counters=ct)
    t, foot, dist = t.cpu().numpy(), foot.cpu().numpy(), dist.cpu().numpy()
    assert ct.cpu().numpy()[L.CNT_PASS2] > 0  # the fallback ran
    o = oracle_lib.project_block(prep.seg_pts, prep.seg_ta, prep.seg_tb, prep.seam_t,
                                 prep.seam_pt, q, workers=8)
    assert np.abs(dist - o["dist"]).max() <= 1e-12
    assert np.abs(t - o["t"]).max() <= 1e-12
    z = np.nonzero(np.all(q == 0.0, axis=1))[0]
    assert np.all(t[z] == 0.0) and np.all(dist[z] == 5.0)


def test_wave_buffer_overflow_falls_back_exactly(gpu):
    """Pair and survivor buffers forced far below the batch's needs
    (MREP_WAVE_PCAP / MREP_WAVE_SCAP): the fused cell-scan filter's staged
    appends, the filter kernel, the pairs kernel and the partitioned clip
    queue all overflow, their queries finish in the fallback kernel, and
    t / foot / distance / segment still equal the dense kernel bit for bit."""
    import os
    import subprocess
    import sys
    code = r"""
import numpy as np, sys
sys.path.insert(0, '.')
from paper_2504_11498_b200 import prepare_curve
from paper_2504_11498_b200.fixtures import random_clamped_curve
cv = random_clamped_curve(np.random.default_rng(0), 7, 400, 3, uniform_knots=True)
tab = prepare_curve(cv, 1e-4).table
q = np.random.default_rng(11).uniform(-0.1, 1.1, (70000, 3))
ra, rb = tab.project(q), tab.project(q, screen=False)
for k in (0, 1, 2, 4):
    a, b = ra[k].cpu().numpy(), rb[k].cpu().numpy()
    assert np.array_equal(a, b), (k, np.nonzero(a != b)[0][:10])
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for caps in ({"MREP_WAVE_PCAP": "20000"}, {"MREP_WAVE_SCAP": "15000"},
                 {"MREP_WAVE_PCAP": "40000", "MREP_WAVE_SCAP": "30000", "MREP_TRAV_FILTER": "1"}):
        env = dict(os.environ, **caps)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           cwd=root, timeout=600)
        assert r.returncode == 0 and "ok" in r.stdout, (caps, r.stderr[-2000:])
