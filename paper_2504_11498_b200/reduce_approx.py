"""G1 cubic reduction and error-controlled approximation on the GPU --
the reference's reduce_approx.py surface.

approximate_error_controlled (reduce_approx.py:207-301) runs entirely in
libmrep (mrep_approx_run): a device FIFO of pending cubics processed in
batches of at most batch_cap, one warp per item for the 64-sample check and
1024-sample verification, exclusive-scan child slots, one warp per child for
the restrict + G1 re-fit + C0 snap, and a final (curve, ta) radix sort.  The
single-item ops (reduce_points_g1, elevate_degree, measure_l1_error,
subdivide_and_modify) call the same device routines.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .core import (
    BezierSegment,
    CubicApproxSegment,
    DepthExceeded,
    DomainError,
    as_readonly,
)


@dataclass(frozen=True, eq=False)
class ReductionSolution:
    """Optimal tangent magnitudes, the resulting cubic and its L2 error."""

    delta0: float
    delta1: float
    cubic: np.ndarray
    l2_error: float

    def __post_init__(self):
        object.__setattr__(self, "cubic", as_readonly(self.cubic))


@dataclass(frozen=True, eq=False)
class SubdivisionLevel:
    """One processed batch: its records, child prefix sums, failing indices."""

    segments: tuple
    child_prefix_sum: np.ndarray
    compaction_keys: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "child_prefix_sum",
                           as_readonly(self.child_prefix_sum, dtype=np.int64))
        object.__setattr__(self, "compaction_keys",
                           as_readonly(self.compaction_keys, dtype=np.int64))


def _pts(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def reduce_points_g1(Q: np.ndarray) -> ReductionSolution:
    """L2-optimal G1 cubic of degree-p control points (p >= 4), on the GPU."""
    Q = _pts(Q)
    p = len(Q) - 1
    if p < 4:
        raise DomainError(f"reduction needs degree >= 4, got {p}")
    d = Q.shape[1]
    Qd = L.to_dev(Q)
    R, delta, l2 = L.empty((4, d)), L.empty((2,)), L.empty((1,))
    L.check(L.lib().mrep_reduce_g1(L.ptr(Qd), p, d, 1, L.ptr(R), L.ptr(delta), L.ptr(l2),
                                   L.stream_ptr()))
    dl = L.to_host(delta)
    return ReductionSolution(float(dl[0]), float(dl[1]), L.to_host(R), float(L.to_host(l2)[0]))


def reduce_to_cubic_g1(segment: BezierSegment) -> ReductionSolution:
    return reduce_points_g1(segment.control_points)


def elevate_degree(segment: BezierSegment, target: int) -> BezierSegment:
    """Same point set at a higher degree (exact, reduce_approx.py:129-143)."""
    if target < segment.degree:
        raise DomainError(f"cannot elevate degree {segment.degree} down to {target}")
    P = _pts(segment.control_points)
    d = P.shape[1]
    Pd = L.to_dev(P)
    out = L.empty((target + 1, d))
    L.check(L.lib().mrep_elevate(L.ptr(Pd), segment.degree, d, int(target), L.ptr(out),
                                 L.stream_ptr()))
    return BezierSegment(target, L.to_host(out), segment.source_interval)


def _max_error(P, approx_iv, Q, orig_iv, samples):
    P, Q = _pts(P), _pts(Q)
    d = P.shape[1]
    Pd, Qd = L.to_dev(P), L.to_dev(Q)
    torch = L._torch()
    mx = L.empty((1,))
    words = (samples + 31) // 32
    mask = L.empty((words,), torch.int32)
    L.check(L.lib().mrep_max_error(L.ptr(Pd), float(approx_iv[0]), float(approx_iv[1]), L.ptr(Qd),
                                   len(Q) - 1, d, float(orig_iv[0]), float(orig_iv[1]),
                                   int(samples), L.ptr(mx), L.ptr(mask), L.stream_ptr()))
    bits = L.to_host(mask).view(np.uint32)
    sel = np.unpackbits(bits.view(np.uint8), bitorder="little")[:samples].astype(bool)
    us = np.linspace(0.0, 1.0, samples)
    return float(L.to_host(mx)[0]), us[sel]


def measure_l1_error(approx: CubicApproxSegment, original: BezierSegment, samples: int = 64):
    """(max error, every local parameter attaining it within 1e-12)."""
    if samples < 2:
        raise DomainError("samples must be >= 2")
    oa, ob = original.source_interval
    aa, ab = approx.source_interval
    if aa < oa - 1e-12 or ab > ob + 1e-12:
        raise DomainError("approximant interval must lie inside the original's")
    return _max_error(approx.control_points, approx.source_interval,
                      original.control_points, original.source_interval, samples)


def subdivide_and_modify(approx: CubicApproxSegment, original: BezierSegment, z: float):
    """Split the cubic at z and snap the shared point onto the original."""
    if not 0.0 < z < 1.0:
        raise DomainError(f"split parameter {z} outside (0, 1)")
    P, Q = _pts(approx.control_points), _pts(original.control_points)
    d = P.shape[1]
    Pd, Qd = L.to_dev(P), L.to_dev(Q)
    Ld, Rd = L.empty((4, d)), L.empty((4, d))
    aa, ab = approx.source_interval
    oa, ob = original.source_interval
    L.check(L.lib().mrep_split_cubic(L.ptr(Pd), d, float(z), 1, aa, ab, L.ptr(Qd), len(Q) - 1,
                                     oa, ob, L.ptr(Ld), L.ptr(Rd), L.stream_ptr()))
    t_split = aa + z * (ab - aa)
    return (CubicApproxSegment(L.to_host(Ld), (aa, t_split), np.inf),
            CubicApproxSegment(L.to_host(Rd), (t_split, ab), np.inf))


class ApproxResult:
    """Device-side cubics of one approximate run, sorted by (curve, ta)."""

    def __init__(self, handle, d):
        self.handle = handle
        self.d = d
        self.count = L.lib().mrep_approx_count(handle)

    def fetch(self):
        torch = L._torch()
        S = self.count
        pts, iv = L.empty((S, 4, self.d)), L.empty((S, 2))
        err, curve = L.empty((S,)), L.empty((S,), torch.int32)
        if S:
            L.check(L.lib().mrep_approx_fetch(self.handle, L.ptr(pts), L.ptr(iv), L.ptr(err),
                                              L.ptr(curve), L.stream_ptr()))
        return pts, iv, err, curve

    def levels(self):
        out = []
        lib = L.lib()
        for lv in range(lib.mrep_approx_num_levels(self.handle)):
            nrec, nfail = ctypes.c_int64(), ctypes.c_int64()
            L.check(lib.mrep_approx_level_sizes(self.handle, lv, ctypes.byref(nrec),
                                                ctypes.byref(nfail)))
            B, F = nrec.value, nfail.value
            P = np.empty((B, 4, self.d))
            iv = np.empty((B, 2))
            err = np.empty(B)
            prefix = np.empty(F + 1, dtype=np.int64)
            keys = np.empty(max(F, 1), dtype=np.int64)
            p = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
            L.check(lib.mrep_approx_level_fetch(self.handle, lv, p(P), p(iv), p(err), p(prefix),
                                                p(keys)))
            recs = tuple(CubicApproxSegment(P[j], (iv[j, 0], iv[j, 1]), err[j]) for j in range(B))
            out.append(SubdivisionLevel(recs, prefix, keys[:F]))
        return out

    def free(self):
        """Release the device buffers now (prepare paths call this right
        after fetch() instead of waiting for garbage collection)."""
        if self.handle:
            L.load_library().mrep_approx_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def approximate_device(rows, row_ofs, iv, curve, nseg, d, tol, batch_cap=4096,
                       loop_samples=64, verify_samples=1024, max_depth=32,
                       collect_levels=False) -> ApproxResult:
    """approximate_error_controlled over device CSR segments (no host copies)."""
    h = ctypes.c_void_p()
    rc = L.lib().mrep_approx_run(L.ptr(rows), L.ptr(row_ofs), L.ptr(iv), L.ptr(curve), int(nseg),
                                 int(d), float(tol), int(batch_cap), int(loop_samples),
                                 int(verify_samples), int(max_depth), int(bool(collect_levels)),
                                 ctypes.byref(h), L.stream_ptr())
    if rc == 3:
        raise DepthExceeded(L.load_library().mrep_last_error().decode())
    L.check(rc)
    return ApproxResult(h, d)


def approximate_error_controlled(segments, tol: float, batch_cap: int = 4096,
                                 loop_samples: int = 64, verify_samples: int = 1024,
                                 max_depth: int = 32, collect_levels: bool = False):
    """Cubics whose max deviation stays <= tol, sorted by source interval.

    Returns (cubics, levels) when collect_levels is set.
    """
    if not tol > 0.0:
        raise DomainError("tolerance must be positive")
    segments = list(segments)
    if not segments:
        return ([], []) if collect_levels else []
    torch = L._torch()
    d = segments[0].control_points.shape[1]
    rows = np.concatenate([_pts(s.control_points) for s in segments])
    lens = [s.control_points.shape[0] for s in segments]
    row_ofs = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    iv = np.array([s.source_interval for s in segments], dtype=np.float64)
    res = approximate_device(L.to_dev(rows), L.to_dev(row_ofs, torch.int64), L.to_dev(iv),
                             None, len(segments), d, tol, batch_cap, loop_samples,
                             verify_samples, max_depth, collect_levels)
    pts, ivs, err, _ = res.fetch()
    pts, ivs, err = L.to_host(pts), L.to_host(ivs), L.to_host(err)
    cubics = [CubicApproxSegment(pts[i], (ivs[i, 0], ivs[i, 1]), float(err[i]))
              for i in range(res.count)]
    levels = res.levels() if collect_levels else None
    res.free()
    return (cubics, levels) if collect_levels else cubics
