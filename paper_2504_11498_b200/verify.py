"""Independent verification helpers -- the reference's oracle.py API surface
(oracle.py:45-160).

eval_de_boor_many / eval_de_boor: Cox-de Boor evaluation (mrep_eval_curve).
oracle_project_batch / oracle_project: dense grid + ternary search on the
GPU (mrep_oracle_project_batch), the CLI's --verify oracle.
decompose_by_knot_insertion / bisect_poly_roots: deliberately naive host
checks for the self-test (they must share no code with the GPU pipeline).
"""

import numpy as np

from . import _lib as L
from .core import BSplineCurve, DomainError


def _basis_rows(knots, p: int, ts) -> np.ndarray:
    """All basis values N_{i,p}(t), one row per t (oracle.py:13-42): half-open
    spans, the right domain end on the final nonzero span."""
    torch = L._torch()
    kn = np.ascontiguousarray(knots, dtype=np.float64)
    ts = np.ascontiguousarray(np.asarray(ts, dtype=np.float64).reshape(-1))
    ncol = len(kn) - 1 - p
    out = torch.zeros((len(ts), max(ncol, 0)), dtype=torch.float64, device=L.device())
    if len(ts) and ncol > 0:
        kd, td = L.to_dev(kn), L.to_dev(ts)
        L.check(L.lib().mrep_basis_rows(int(p), L.ptr(kd), len(kn), L.ptr(td), len(ts), L.ptr(out),
                                        L.stream_ptr()))
    return L.to_host(out)


def eval_de_boor_many(curve: BSplineCurve, ts) -> np.ndarray:
    """Curve points at an array of parameters (oracle.py:45-52)."""
    ts = np.ascontiguousarray(np.asarray(ts, dtype=np.float64).reshape(-1))
    lo, hi = curve.domain
    if np.any(ts < lo) or np.any(ts > hi):
        raise DomainError(f"parameter outside domain [{lo}, {hi}]")
    d = curve.dimension
    kn = L.to_dev(curve.knots.knots)
    cp = L.to_dev(curve.control_points)
    td = L.to_dev(ts)
    out = L.empty((len(ts), d))
    if len(ts):
        L.check(L.lib().mrep_eval_curve(curve.degree, L.ptr(kn), len(curve.knots.knots),
                                        L.ptr(cp), curve.control_points.shape[0], d, L.ptr(td),
                                        len(ts), L.ptr(out), L.stream_ptr()))
    return L.to_host(out)


def eval_de_boor(curve: BSplineCurve, t: float) -> np.ndarray:
    return eval_de_boor_many(curve, [t])[0]


def oracle_project_batch(curve: BSplineCurve, queries, grid: int = 4096):
    """Brute-force nearest parameter for many queries (oracle.py:95-128) on
    the GPU: dense scan of `grid` curve points, then ternary search on each
    query's bracketing cells down to width 1e-10.  Returns
    (t, distance, resolution); resolution is the largest distance between
    adjacent grid points (oracle.py:108)."""
    if grid < 2:
        raise DomainError("grid must be >= 2")
    q = np.ascontiguousarray(np.atleast_2d(np.asarray(queries, dtype=np.float64)))
    lo, hi = curve.domain
    ts = np.linspace(lo, hi, grid)
    pts = eval_de_boor_many(curve, ts)
    resolution = float(np.linalg.norm(np.diff(pts, axis=0), axis=1).max())
    n = len(q)
    if n == 0:
        return np.empty(0), np.empty(0), resolution
    d = curve.dimension
    kn = L.to_dev(curve.knots.knots)
    cp = L.to_dev(curve.control_points)
    tsd, ptsd, qd = L.to_dev(ts), L.to_dev(pts), L.to_dev(q)
    t_out, d_out = L.empty((n,)), L.empty((n,))
    L.check(L.lib().mrep_oracle_project_batch(
        curve.degree, L.ptr(kn), len(curve.knots.knots), L.ptr(cp),
        curve.control_points.shape[0], d, L.ptr(tsd), L.ptr(ptsd), grid, L.ptr(qd), n,
        L.ptr(t_out), L.ptr(d_out), L.stream_ptr()))
    return L.to_host(t_out), L.to_host(d_out), resolution


def oracle_project(curve: BSplineCurve, q, grid: int = 4096):
    """Single-query wrapper (oracle.py:131-134)."""
    t, d, res = oracle_project_batch(curve, [q], grid)
    return float(t[0]), float(d[0]), res


# ---- independent host-side checks (selftest / tests only; not the hot path)
def decompose_by_knot_insertion(curve: BSplineCurve):
    """Classical serial decomposition by Boehm knot insertion, every interior
    knot raised to multiplicity p (oracle.py:59-92) -- an independent check of
    the matrix decomposition, deliberately sharing no code with it."""
    from .core import BezierSegment, validate_curve
    validate_curve(curve)
    p = curve.degree
    knots = np.array(curve.knots.knots, dtype=np.float64)
    cp = np.array(curve.control_points, dtype=np.float64)
    lo, hi = curve.domain
    for t in sorted(set(knots[(knots > lo) & (knots < hi)])):
        while np.count_nonzero(knots == t) < p:
            k = int(np.searchsorted(knots, t, side="right")) - 1
            new = np.empty((len(cp) + 1, cp.shape[1]))
            for i in range(len(cp) + 1):
                if i <= k - p:
                    new[i] = cp[i]
                elif i <= k:
                    a = (t - knots[i]) / (knots[i + p] - knots[i])
                    new[i] = (1.0 - a) * cp[i - 1] + a * cp[i]
                else:
                    new[i] = cp[i - 1]
            knots, cp = np.insert(knots, k + 1, t), new
    breaks = sorted(set(knots))
    segs, start = [], 0
    for i in range(len(breaks) - 1):
        segs.append(BezierSegment(p, cp[start: start + p + 1], (breaks[i], breaks[i + 1])))
        start += p
    return segs


def bisect_poly_roots(coeffs, lo: float = 0.0, hi: float = 1.0, cells: int = 4096,
                      tol: float = 1e-9) -> np.ndarray:
    """Sign-change scan + bisection (oracle.py:137-160): the reference for
    the closed-form quartic solver in the self-test."""
    c = np.asarray(coeffs, dtype=np.float64)[::-1]
    ts = np.linspace(lo, hi, cells + 1)
    vals = np.polyval(c, ts)
    roots = [float(t) for t, v in zip(ts, vals) if v == 0.0]
    idx = np.nonzero(vals[:-1] * vals[1:] < 0.0)[0]
    a, b, fa = ts[idx].copy(), ts[idx + 1].copy(), vals[idx].copy()
    while len(a) and np.max(b - a) > tol:
        m = 0.5 * (a + b)
        fm = np.polyval(c, m)
        left = fa * fm <= 0.0
        b = np.where(left, m, b)
        a = np.where(left, a, m)
        fa = np.where(left, fa, fm)
    roots.extend((0.5 * (a + b)).tolist())
    out = []
    for r in sorted(roots):
        if not out or r - out[-1] > 1e-10:
            out.append(r)
    return np.array(out)
