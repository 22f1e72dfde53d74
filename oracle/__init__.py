"""CPU ORACLE -- test infrastructure only.

Two restatements of the reference (`/root/reference/pkg/src/splinemat`):

* ``mrep_oracle.c`` (loaded here through ctypes): the numba per-query kernels
  of ``_kernels.py``, bit-for-bit on the same libm, multi-threaded with OpenMP
  the way ``project.py:266-281`` fans out over threads.
* ``mrep_surface_oracle.c``: the surface projection (the reference has none;
  this file defines the algorithm the GPU implements, brute force over every
  patch) and ``surface.py``: numpy surface decomposition + a dense-grid
  global search that checks the minimiser is global.
* ``prep.py``: the numpy preprocessing of ``basis.py`` / ``decompose.py`` /
  ``reduce_approx.py`` (decomposition and error-controlled cubic
  approximation), same numpy expressions, so it matches the reference
  bit-for-bit on the same BLAS.

Pinned against the reference's own outputs in ``tests/golden`` (see
``tests/test_oracle_pin.py``).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (its CPU-baseline leg and ``--impl reference``) may import
this package; the product package never does.
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libmrep_oracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)


def build():
    """Compile the C oracle in place (gcc, no GPU needed)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        srcs = [os.path.join(_HERE, f) for f in ("mrep_oracle.c", "mrep_surface_oracle.c")]
        if not os.path.exists(_LIB_PATH) or any(
                os.path.getmtime(_LIB_PATH) < os.path.getmtime(f) for f in srcs):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_quartic_roots_01.argtypes = [_dp, _dp]
        L.oracle_quartic_roots_01.restype = ctypes.c_int
        L.oracle_distance_poly.argtypes = [_dp, ctypes.c_int, _dp, _dp]
        L.oracle_restrict_ordinates.argtypes = [_dp, ctypes.c_double, ctypes.c_double, _dp]
        L.oracle_eval_ordinates.argtypes = [_dp, ctypes.c_double]
        L.oracle_eval_ordinates.restype = ctypes.c_double
        L.oracle_hull_cross.argtypes = [_dp, _dp, _dp]
        L.oracle_hull_cross.restype = ctypes.c_int
        L.oracle_clip_root.argtypes = [_dp, ctypes.c_double, ctypes.c_int, _dp,
                                       ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
        L.oracle_clip_root.restype = ctypes.c_double
        L.oracle_decasteljau_point.argtypes = [_dp, ctypes.c_int, ctypes.c_double, _dp]
        L.oracle_project_block.argtypes = [
            _dp, _dp, _dp, _dp, _dp, ctypes.c_int64, ctypes.c_int, _dp, ctypes.c_int64,
            ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            _dp, _dp, _dp, _i64p, _i64p, _dp, _i64p, _i32p, _i32p]
        L.oracle_quartic_block.argtypes = [_dp, ctypes.c_int64, _dp, _i64p]
        L.oracle_newton_quartic_block.argtypes = [_dp, ctypes.c_int64, _dp, _i64p]
        L.oracle_surf_patch_min.argtypes = [_dp, ctypes.c_int, ctypes.c_int, _dp, _dp, _dp, _dp,
                                            ctypes.POINTER(ctypes.c_int)]
        L.oracle_surface_project.argtypes = [_dp, _dp, ctypes.c_int64, ctypes.c_int,
                                             ctypes.c_int, _dp, ctypes.c_int64, ctypes.c_int,
                                             _dp, _dp, _dp, _dp, _i32p, _i32p]
        _lib = L
    return _lib


def _p(a, t=_dp):
    return a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def quartic_roots_01(c):
    c = _f64(c)
    out = np.zeros(4)
    n = lib().oracle_quartic_roots_01(_p(c), _p(out))
    return out[:n].copy()


def quartic_block(coeffs):
    coeffs = _f64(coeffs)
    n = coeffs.shape[0]
    roots = np.full((n, 4), np.nan)
    counts = np.zeros(n, dtype=np.int64)
    lib().oracle_quartic_block(_p(coeffs), n, _p(roots), _p(counts, _i64p))
    return roots, counts


def newton_quartic_block(coeffs):
    coeffs = _f64(coeffs)
    n = coeffs.shape[0]
    roots = np.full((n, 4), np.nan)
    counts = np.zeros(n, dtype=np.int64)
    lib().oracle_newton_quartic_block(_p(coeffs), n, _p(roots), _p(counts, _i64p))
    return roots, counts


def distance_poly(P, q):
    P = _f64(P)
    q = _f64(q)
    e = np.zeros(6)
    lib().oracle_distance_poly(_p(P), P.shape[1], _p(q), _p(e))
    return e


def restrict_ordinates(b, lo, hi):
    b = _f64(b)
    out = np.zeros(6)
    lib().oracle_restrict_ordinates(_p(b), float(lo), float(hi), _p(out))
    return out


def eval_ordinates(b, u):
    b = _f64(b)
    return lib().oracle_eval_ordinates(_p(b), float(u))


def hull_cross(b):
    b = _f64(b)
    z1 = ctypes.c_double()
    z2 = ctypes.c_double()
    f = lib().oracle_hull_cross(_p(b), ctypes.byref(z1), ctypes.byref(z2))
    return bool(f), z1.value, z2.value


def clip_root(b, tol, max_iter):
    b = _f64(b)
    w = np.zeros(max(max_iter, 1))
    ok = ctypes.c_int()
    used = ctypes.c_int()
    r = lib().oracle_clip_root(_p(b), float(tol), int(max_iter), _p(w),
                               ctypes.byref(ok), ctypes.byref(used))
    return r, bool(ok.value), used.value, w[:max_iter]


def decasteljau_point(P, u):
    P = _f64(P)
    out = np.zeros(P.shape[1])
    lib().oracle_decasteljau_point(_p(P), P.shape[1], float(u), _p(out))
    return out


def project_block(seg_pts, seg_ta, seg_tb, seam_t, seam_pt, queries, clip_tol=1e-6,
                  max_iter=8, soundness_samples=0, workers=1):
    """The reference's _project_block over a query batch (workers = OpenMP threads).

    Returns dict(t, foot, dist, cand, stats[n,6], sound, win, seg, tie); tie[i]
    counts candidates of another segment within dmin + 2e-12 (query i's
    winning segment is ambiguous at the ulp level iff tie[i] > 0)."""
    seg_pts, seg_ta, seg_tb = _f64(seg_pts), _f64(seg_ta), _f64(seg_tb)
    seam_t, seam_pt, queries = _f64(seam_t), _f64(seam_pt), _f64(np.atleast_2d(queries))
    S, _, d = seg_pts.shape
    n = queries.shape[0]
    out = dict(t=np.empty(n), foot=np.empty((n, d)), dist=np.empty(n),
               cand=np.empty(n, dtype=np.int64), stats=np.zeros((n, 6), dtype=np.int64),
               sound=np.empty(n), win=np.empty(n, dtype=np.int64),
               seg=np.empty(n, dtype=np.int32), tie=np.empty(n, dtype=np.int32))
    lib().oracle_project_block(
        _p(seg_pts), _p(seg_ta), _p(seg_tb), _p(seam_t), _p(seam_pt), S, d, _p(queries), n,
        float(clip_tol), int(max_iter), int(soundness_samples), int(workers),
        _p(out["t"]), _p(out["foot"]), _p(out["dist"]), _p(out["cand"], _i64p),
        _p(out["stats"], _i64p), _p(out["sound"]), _p(out["win"], _i64p),
        _p(out["seg"], _i32p), _p(out["tie"], _i32p))
    return out


def surface_project(patch_pts, patch_iv, pu, pv, queries, workers=1):
    """Brute-force surface projection (mrep_surface_oracle.c): patch_pts
    [np][pu+1][pv+1][3] and patch_iv [np][4] in patch-id order.
    Returns dict(u, v, foot, dist, patch, tie); tie = another patch's
    minimum within dmin (1 + 1e-9) + 1e-12 (the winner then rests on
    rounding-level differences)."""
    P = _f64(patch_pts).reshape(-1)
    I = _f64(patch_iv).reshape(-1)
    q = _f64(np.atleast_2d(queries))
    npat = P.size // ((pu + 1) * (pv + 1) * 3)
    n = q.shape[0]
    out = dict(u=np.empty(n), v=np.empty(n), foot=np.empty((n, 3)), dist=np.empty(n),
               patch=np.empty(n, dtype=np.int32), tie=np.empty(n, dtype=np.int32))
    lib().oracle_surface_project(_p(P), _p(I), npat, pu, pv, _p(q), n, int(workers),
                                 _p(out["u"]), _p(out["v"]), _p(out["foot"]), _p(out["dist"]),
                                 _p(out["patch"], _i32p), _p(out["tie"], _i32p))
    return out


def surf_patch_min(P, pu, pv, q):
    """(u, v, d2, iters) of one patch (local parameters)."""
    P = _f64(P).reshape(-1)
    q = _f64(q)
    u, v, d2, it = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
    lib().oracle_surf_patch_min(_p(P), pu, pv, _p(q), ctypes.byref(u), ctypes.byref(v),
                                ctypes.byref(d2), ctypes.byref(it))
    return u.value, v.value, d2.value, it.value
