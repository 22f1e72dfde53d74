"""Batch point projection and inversion on the B200 -- the reference's
project.py surface (project.py:40-348), same names, arguments, return
types and errors.

prepare_curve runs decomposition + error-controlled approximation on the GPU
and keeps the packed segment table (plus its AABB hierarchy) resident in HBM
inside the returned PreparedCurve; project_prepared ships the queries to the
device, runs the sm_100a projection kernel and returns host arrays, exactly
like the reference's numba batch driver.

Modes of project_prepared:
* default (screen=True, cand="exact"): BVH-screened exact solve.  t, foot,
  distance (and the winning segment) are those of the brute-force reference
  kernel; `cand` is the reference's own count -- every seam plus every
  surviving piece of every cubic -- computed by a separate pass on the FP64
  tensor cores (one mma.sync m8n8k4 per 8 queries x 1 cubic decides the sign
  of E' on each cubic; the few undecided pairs are solved exactly;
  csrc/mrep_cand.cuh).
* cand="screened": skip that pass; `cand` then counts what the query's
  screened traversal examined (seams offered plus cubics queued for the
  exact solve) -- the fast path the C-ABI benchmark measures.
* screen=False, or with_stats / soundness_samples: brute force over all
  cubics with the reference's exact cand, ProjectionStats and soundness.
`workers` is accepted and validated (plan_work) for drop-in compatibility;
results never depend on it.
"""

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib as L
from .basis import power_to_bernstein_matrix  # noqa: F401  (re-exported helper parity)
from .core import (
    BSplineCurve,
    CubicApproxSegment,
    DomainError,
    NoRoot,
    Poly,
    PointNotOnCurve,
    ProjectionResult,
    as_readonly,
    eval_bezier,
)
from .decompose import DeviceCurves, decompose_device
from .core import EmptyDomain, validate_curve
from .distance import distance_polys, monotonic_split
from .reduce_approx import approximate_device


@dataclass(frozen=True, eq=False)
class NonParametricBezier:
    """Scalar quintic in Bernstein form: ordinates b_i at abscissae i/5."""

    ordinates: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "ordinates", as_readonly(self.ordinates))

    @property
    def degree(self) -> int:
        return len(self.ordinates) - 1

    @property
    def e_start(self) -> float:
        return float(self.ordinates[0])

    @property
    def e_end(self) -> float:
        return float(self.ordinates[-1])

    def __call__(self, u: float) -> float:
        if _quintic(self):
            return float(D.eval_ordinates(self.ordinates[None], float(u))[0])
        return float(D.ordinates_op(0, self.ordinates[None], a=float(u))[0])


def _quintic(bez):
    """Quintic E (the only degree the projection builds) -> the fixed-size
    kernels the projection itself runs; any other degree (1..31) -> the
    runtime-degree kernels (mrep_ordinates_op)."""
    n = len(bez.ordinates)
    if n < 2 or n > 32:
        raise DomainError("ordinate ops need degree 1..31")
    return n == 6


@dataclass(frozen=True, eq=False)
class PieceCandidate:
    segment: CubicApproxSegment
    ordinates: NonParametricBezier


@dataclass(frozen=True, eq=False)
class CandidateSet:
    endpoints: tuple
    pieces: tuple


@dataclass(frozen=True)
class WorkPlan:
    total_units: int
    workers: int
    units_per_worker: int


@dataclass(frozen=True, eq=False)
class ClipResult:
    root: float
    width: float
    iterations: int
    converged_at: int | None


@dataclass(frozen=True, eq=False)
class ProjectionStats:
    pieces: int
    conv3_local: int
    conv3_source: int
    conv_final_local: int
    conv_final_source: int
    hull_misses: int


class PreparedCurve:
    """Per-curve arrays (host, read-only) + the device-resident segment table.

    Fields match the reference dataclass (project.py:110-121); `cubics` is
    materialised lazily because curve sets reach 10^5 cubics.
    """

    def __init__(self, curve, tolerance, seg_pts, seg_ta, seg_tb, seam_t, seam_pt,
                 measured_error=None, table=None, cubics=None):
        self.curve = curve
        self.tolerance = tolerance
        self.seg_pts = as_readonly(seg_pts)
        self.seg_ta = as_readonly(seg_ta)
        self.seg_tb = as_readonly(seg_tb)
        self.seam_t = as_readonly(seam_t)
        self.seam_pt = as_readonly(seam_pt)
        self._err = None if measured_error is None else as_readonly(measured_error)
        self._table = table
        self._cubics = cubics

    @classmethod
    def from_arrays(cls, curve, tolerance, seg_pts, seg_ta, seg_tb, seam_t, seam_pt, cubics=None):
        """Wrap already-packed arrays (e.g. a reference PreparedCurve's fields)."""
        return cls(curve, tolerance, seg_pts, seg_ta, seg_tb, seam_t, seam_pt, cubics=cubics)

    @property
    def cubics(self):
        if self._cubics is None:
            err = self._err if self._err is not None else np.zeros(len(self.seg_ta))
            self._cubics = tuple(
                CubicApproxSegment(self.seg_pts[i], (self.seg_ta[i], self.seg_tb[i]), float(err[i]))
                for i in range(len(self.seg_ta)))
        return self._cubics

    @property
    def table(self) -> D.DeviceTable:
        if self._table is None:
            self._table = D.DeviceTable(self.seg_pts, self.seg_ta, self.seg_tb, self.seam_t,
                                        self.seam_pt)
        return self._table

    @property
    def num_segments(self) -> int:
        return len(self.seg_ta)

    def knot_spans(self, t):
        """Knot span of each parameter on the GPU (mrep_knot_span):
        searchsorted(knots, t, 'right') - 1 clipped to [p, n - 1], the span
        convention of core.py:108-112.  t: host array or device tensor."""
        torch = L._torch()
        if self.curve is None:
            raise DomainError("knot spans need the prepared curve's knot vector")
        if getattr(self, "_knots_dev", None) is None:
            self._knots_dev = L.to_dev(np.asarray(self.curve.knots.knots, dtype=np.float64))
        td = L.to_dev(t)
        n = int(td.shape[0])
        span = torch.empty((n,), dtype=torch.int32, device=td.device)
        L.check(L.lib().mrep_knot_span(L.ptr(self._knots_dev), int(self._knots_dev.shape[0]),
                                       int(self.curve.degree), L.ptr(td), n, L.ptr(span),
                                       L.stream_ptr()))
        return L.to_host(span)


# ------------------------------------------------------------ single-pair ops
def rebase(e) -> NonParametricBezier:
    """Power coefficients (degree <= 5) -> Bernstein ordinates (T5 e)."""
    coeffs = e.coeffs if isinstance(e, Poly) else np.asarray(e, dtype=np.float64)
    if len(coeffs) > 6 and np.any(coeffs[6:] != 0.0):
        raise DomainError("rebase expects degree <= 5")
    c = np.zeros(6)
    c[: min(6, len(coeffs))] = coeffs[:6]
    return NonParametricBezier(D.rebase(c[None])[0])


def rebase_batch(coeff_block: np.ndarray) -> np.ndarray:
    """Rebase many coefficient rows (n, 6) at once."""
    block = np.asarray(coeff_block, dtype=np.float64)
    return D.rebase(block.reshape(-1, 6)).reshape(block.shape)


def hull_x_intersections(bez: NonParametricBezier):
    """Abscissa range where the convex hull meets y = 0, or None."""
    found, z = (D.hull_cross if _quintic(bez) else
                lambda b: D.ordinates_op(1, b))(bez.ordinates[None])
    return (float(z[0, 0]), float(z[0, 1])) if found[0] else None


def clip(bez: NonParametricBezier, z1: float, z2: float) -> NonParametricBezier:
    """Restrict to [z1, z2] (project.py:146-156), de Casteljau on the GPU."""
    if not 0.0 <= z1 <= z2 <= 1.0:
        raise DomainError(f"bad clip interval [{z1}, {z2}]")
    quintic = _quintic(bez)
    b = np.asarray(bez.ordinates)
    if z1 >= 1.0:
        return NonParametricBezier(np.full(len(b), b[-1]))
    if quintic:
        return NonParametricBezier(D.restrict_ordinates(b[None], z1, z2)[0])
    return NonParametricBezier(D.ordinates_op(2, b[None], a=z1, c=z2)[0])


def clip_root(bez: NonParametricBezier, tol: float = 1e-6,
              max_iterations: int = 8) -> ClipResult:
    """Bezier clipping of an eliminated piece down to width tol."""
    quintic = _quintic(bez)
    if max_iterations < 1:
        raise DomainError("max_iterations must be >= 1")
    if quintic:
        root, ok, used, widths = D.clip_root(bez.ordinates[None], tol, max_iterations)
    else:
        root, ok, used, widths = D.ordinates_op(3, bez.ordinates[None], tol=tol,
                                                max_iter=max_iterations)
    if not ok[0]:
        raise NoRoot("convex hull never crosses the axis")
    used = int(used[0])
    w = widths[0]
    conv = next((k + 1 for k in range(used) if w[k] <= tol), None)
    return ClipResult(float(root[0]), float(w[used - 1]), used, conv)


def eliminate(pieces, start_candidate, end_candidate) -> CandidateSet:
    """Keep pieces with E(0) < 0 and E(0) E(1) <= 0; attach both endpoints."""
    kept = tuple(pc for pc in pieces
                 if pc.ordinates.e_start < 0.0
                 and pc.ordinates.e_start * pc.ordinates.e_end <= 0.0)
    return CandidateSet((start_candidate, end_candidate), kept)


def reduce_min(query, candidates) -> ProjectionResult:
    """Smallest distance, ties within 1e-12 broken by smallest t (two passes)."""
    cands = list(candidates)
    if not cands:
        raise DomainError("reduce_min needs at least the endpoint candidates")
    dmin = min(d for _, _, d in cands)
    best = min((t, i) for i, (t, _, d) in enumerate(cands) if d <= dmin + 1e-12)[1]
    t, foot, dist = cands[best]
    return ProjectionResult(np.asarray(query, dtype=np.float64), float(t),
                            np.asarray(foot, dtype=np.float64), float(dist), len(cands))


def plan_work(total_units: int, workers: int) -> WorkPlan:
    """K = ceil(total / workers) (project.py:212-217)."""
    if workers < 1:
        raise DomainError("workers must be >= 1")
    return WorkPlan(total_units, workers, max(1, -(-total_units // workers)))


# ------------------------------------------------------------ preparation
def _pack_device(pts, iv, err, curve, tolerance):
    """Device cubics of one curve -> PreparedCurve with its resident table."""
    torch = L._torch()
    ta = iv[:, 0].contiguous()
    tb = iv[:, 1].contiguous()
    seam_t = torch.cat([ta[:1], tb]).contiguous()
    seam_pt = torch.cat([pts[:1, 0, :], pts[:, 3, :]]).contiguous()
    table = D.DeviceTable(pts, ta, tb, seam_t, seam_pt)
    return PreparedCurve(curve, tolerance, L.to_host(pts), L.to_host(ta), L.to_host(tb),
                         L.to_host(seam_t), L.to_host(seam_pt), measured_error=L.to_host(err),
                         table=table)


def prepare_curves(curves, tolerance: float = 1e-4, batch_cap: int = 4096):
    """prepare_curve for many curves in one batched decomposition + approximation."""
    curves = list(curves)
    for c in curves:
        validate_curve(c)
        if not c.span_indices():
            raise EmptyDomain("curve has no nonzero-length span")
    out = [None] * len(curves)
    for d in (2, 3):
        idx = [i for i, c in enumerate(curves) if c.dimension == d]
        if not idx:
            continue
        batch = [curves[i] for i in idx]
        dec = decompose_device(DeviceCurves(batch))
        res = approximate_device(dec["rows"], dec["row_ofs"], dec["iv"], dec["curve"],
                                 dec["nseg"], d, tolerance, batch_cap)
        pts, iv, err, cid = res.fetch()
        res.free()
        cid_h = L.to_host(cid)
        bounds = np.searchsorted(cid_h, np.arange(len(batch) + 1))
        for j, i in enumerate(idx):
            a, b = bounds[j], bounds[j + 1]
            out[i] = _pack_device(pts[a:b], iv[a:b], err[a:b], curves[i], tolerance)
    return out


def prepare_curve(curve: BSplineCurve, tolerance: float = 1e-4,
                  batch_cap: int = 4096) -> PreparedCurve:
    """Decompose and approximate once on the GPU; keep the table resident."""
    return prepare_curves([curve], tolerance, batch_cap)[0]


# ------------------------------------------------------------ projection
def _as_queries(prep, queries):
    q = np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float64)
    if q.shape[1] != prep.curve.dimension:
        raise DomainError("query dimension does not match the curve")
    return q


def project_prepared(prep: PreparedCurve, queries, workers: int | None = None,
                     clip_tol: float = 1e-6, max_iterations: int = 8,
                     with_stats: bool = False, soundness_samples: int = 0, *,
                     screen: bool = True, return_segments: bool = False,
                     return_spans: bool = False, cand: str = "exact"):
    """Project every query; returns (t, foot, distance, candidates) host arrays,
    plus (ProjectionStats, sound) when with_stats, plus the winning cubic index
    per query when return_segments, plus the knot span of t* in the original
    B-spline (core.py:108-112) when return_spans.  cand="exact" (default)
    returns the reference's candidate count, cand="screened" the screened
    traversal's (faster; see the module docstring)."""
    q = _as_queries(prep, queries)
    plan_work(len(q), 1 if workers is None else workers)
    if max_iterations < 1:
        raise DomainError("max_iterations must be >= 1")
    if cand not in ("exact", "screened"):
        raise DomainError('cand must be "exact" or "screened"')
    n = q.shape[0]
    dense = with_stats or soundness_samples > 0 or not screen
    tab = prep.table
    if n == 0:
        empty = (np.empty(0), np.empty((0, q.shape[1])), np.empty(0), np.empty(0, np.int64))
        if with_stats:
            empty = empty + (ProjectionStats(0, 0, 0, 0, 0, 0), np.empty(0))
        return (empty + ((np.empty(0, np.int32),) if return_segments else ())
                + ((np.empty(0, np.int32),) if return_spans else ()))
    if not dense:
        cnt = np.zeros(L.NUM_COUNTERS, dtype=np.uint64)
        t, foot, dist, cnd, seg = tab.project_host(
            q, clip_tol=clip_tol, max_iter=max_iterations, screen=True, counters=cnt,
            extra_flags=L.MREP_CAND_EXACT if cand == "exact" else 0)
        if int(cnt[L.CNT_HULL_MISS]) > 0:
            raise NoRoot("hull never crossed on a surviving piece; elimination bug")
        out = (t, foot, dist, cnd)
        return (out + ((seg,) if return_segments else ())
                + ((prep.knot_spans(t),) if return_spans else ()))
    td, fd, dd, cd, sd, std, snd = tab.project(L.to_dev(q), clip_tol, max_iterations,
                                               soundness_samples, screen=False, stats=True)
    t, foot, dist, cand = L.to_host(td), L.to_host(fd), L.to_host(dd), L.to_host(cd)
    stats_arr, sound, seg = L.to_host(std), L.to_host(snd), L.to_host(sd)
    if int(stats_arr[:, 5].sum()) > 0:
        raise NoRoot("hull never crossed on a surviving piece; elimination bug")
    out = (t, foot, dist, cand)
    if with_stats:
        tot = stats_arr.sum(axis=0)
        out = out + (ProjectionStats(*(int(x) for x in tot)), sound)
    return (out + ((seg,) if return_segments else ())
            + ((prep.knot_spans(td),) if return_spans else ()))


def project_points(curve: BSplineCurve, queries, tolerance: float = 1e-4,
                   workers: int | None = None) -> list[ProjectionResult]:
    """Prepare, project, and wrap each query in a ProjectionResult."""
    if not tolerance > 0.0:
        raise DomainError("tolerance must be positive")
    prep = prepare_curve(curve, tolerance)
    queries = np.atleast_2d(np.asarray(queries, dtype=np.float64))
    t, foot, dist, cand = project_prepared(prep, queries, workers=workers)
    return [ProjectionResult(queries[i], float(t[i]), foot[i], float(dist[i]), int(cand[i]))
            for i in range(len(queries))]


def invert_point(curve: BSplineCurve, q, tolerance: float = 1e-4) -> float:
    """Parameter of a point on the curve; PointNotOnCurve beyond 10 * tolerance."""
    res = project_points(curve, [q], tolerance)[0]
    if res.distance > 10.0 * tolerance:
        raise PointNotOnCurve(
            f"projection distance {res.distance:.3e} exceeds 10 * {tolerance}")
    return res.t_star


def invert_points(prep: PreparedCurve, points, tolerance: float | None = None):
    """Batch inversion against a prepared curve (the path criterion 3 uses):
    parameters of on-curve points; PointNotOnCurve if any lies beyond
    10 * tolerance."""
    tol = prep.tolerance if tolerance is None else tolerance
    t, _, dist, _ = project_prepared(prep, points, cand="screened")
    bad = np.nonzero(dist > 10.0 * tol)[0]
    if len(bad):
        raise PointNotOnCurve(f"{len(bad)} points farther than 10 * {tol} "
                              f"(max {dist[bad].max():.3e})")
    return t


def project_single_reference(prep: PreparedCurve, q) -> ProjectionResult:
    """Single-query projection assembled from the public per-op API
    (monotone split, rebase, eliminate, clip, reduce) -- an independent route
    against the fused batch kernel (project.py:315-343)."""
    q = np.asarray(q, dtype=np.float64)
    start = (float(prep.seam_t[0]), prep.seam_pt[0])
    end = (float(prep.seam_t[-1]), prep.seam_pt[-1])
    pieces = []
    for cub in prep.cubics:
        for piece in monotonic_split(cub, q):
            polys = distance_polys(piece, q)
            pieces.append(PieceCandidate(piece, rebase(polys.e)))
    cset = eliminate(pieces, start, end)
    candidates = [(t, pt, float(np.linalg.norm(q - pt))) for t, pt in cset.endpoints]
    for s in range(1, len(prep.seam_t) - 1):
        pt = prep.seam_pt[s]
        candidates.append((float(prep.seam_t[s]), pt, float(np.linalg.norm(q - pt))))
    for pc in cset.pieces:
        res = clip_root(pc.ordinates)
        ta, tb = pc.segment.source_interval
        foot = eval_bezier(pc.segment.control_points, res.root)
        candidates.append((ta + res.root * (tb - ta), foot, float(np.linalg.norm(q - foot))))
    return reduce_min(q, candidates)


def engine_info() -> dict:
    lib = L.load_library()
    return {"backend": "libmrep-sm_100a", "version": lib.mrep_version()}
