"""Many curves at once: one prepared curve SET, one projection batch in which
every query names its curve (BASELINE.json configs[2], the load-balance
stress case).

The reference has no multi-curve projection call: a user prepares each curve
(prepare_curve, project.py:220-242; batched_decompose, decompose.py:49-67, for
the decomposition) and calls project_prepared per curve
(project.py:245-289).  Here the whole set is decomposed and approximated in
one batched device run, packed into ONE device allocation of per-curve
segment tables (mrep_curveset_create_dev), and projected in ONE call
(mrep_project_batch) whose scheduler sorts queries by (curve, Morton code),
heaviest curve first, and drains them with persistent traversal warps pulling
from an atomic task queue -- the paper's segment-count sorting + persistent
work queue.  Per query, t / foot / dist / segment equal what project_prepared
returns for that query's curve alone.
"""

import ctypes

import numpy as np

from . import _lib as L
from .core import DomainError, EmptyDomain, GeometryError, NoRoot, validate_curve
from .decompose import DeviceCurves, decompose_device
from .project import PreparedCurve, plan_work
from .reduce_approx import approximate_device


class PreparedCurveSet:
    """Prepared cubics of many curves (host arrays, read-only) + the device set.

    seg_pts / seg_ta / seg_tb are the PreparedCurve arrays of every curve
    concatenated in curve order; curve c owns rows seg_ofs[c]:seg_ofs[c+1].
    ``set[c]`` is that curve's PreparedCurve (identical arrays to
    prepare_curve(curves[c])).
    """

    def __init__(self, curves, tolerance, seg_pts, seg_ta, seg_tb, seg_ofs, handle, err=None,
                 dev_curves=None):
        # seg_* / err: numpy arrays, or device tensors fetched to the host on
        # first access (a cfg3 set is ~400 MB of cubics; the device set does
        # not need the host copy)
        self.curves = list(curves)
        self.tolerance = tolerance
        self._arrays = {"seg_pts": seg_pts, "seg_ta": seg_ta, "seg_tb": seg_tb,
                        "measured_error": err}
        self.seg_ofs = np.asarray(seg_ofs, dtype=np.int64)
        self.seg_ofs.flags.writeable = False
        self._handle = handle
        self._dev_curves = dev_curves  # CSR device knots for knot_spans
        self.d = int(seg_pts.shape[2]) if len(seg_pts.shape) == 3 else 3

    def _host(self, name):
        a = self._arrays[name]
        if a is not None and not isinstance(a, np.ndarray):
            a = L.to_host(a)
            a.flags.writeable = False
            self._arrays[name] = a
        elif isinstance(a, np.ndarray) and a.flags.writeable:
            a.flags.writeable = False
        return a

    seg_pts = property(lambda self: self._host("seg_pts"))
    seg_ta = property(lambda self: self._host("seg_ta"))
    seg_tb = property(lambda self: self._host("seg_tb"))
    measured_error = property(lambda self: self._host("measured_error"))

    @property
    def handle(self):
        if self._handle is None:
            raise RuntimeError("curve set was freed")
        return self._handle

    def __len__(self):
        return len(self.curves)

    @property
    def num_segments(self):
        return int(self.seg_ofs[-1])

    def segment_counts(self):
        return np.diff(self.seg_ofs)

    def __getitem__(self, c) -> PreparedCurve:
        a, b = int(self.seg_ofs[c]), int(self.seg_ofs[c + 1])
        pts, ta, tb = self.seg_pts[a:b], self.seg_ta[a:b], self.seg_tb[a:b]
        seam_t = np.concatenate(([ta[0]], tb))
        seam_pt = np.concatenate((pts[:1, 0, :], pts[:, 3, :]))
        err = None if self.measured_error is None else self.measured_error[a:b]
        return PreparedCurve(self.curves[c], self.tolerance, pts, ta, tb, seam_t, seam_pt,
                             measured_error=err)

    def knot_spans(self, t, curve_ids):
        """Knot span of t[i] in curve curve_ids[i] (mrep_knot_span_batch; the
        span convention of core.py:108-112).  Host arrays or device tensors."""
        torch = L._torch()
        if self._dev_curves is None:
            if any(c is None for c in self.curves):
                raise DomainError("knot spans need every curve's knot vector")
            self._dev_curves = DeviceCurves(self.curves)
        dc = self._dev_curves
        td = L.to_dev(t)
        cid = L.to_dev(curve_ids, torch.int32)
        n = int(td.shape[0])
        span = torch.empty((n,), dtype=torch.int32, device=td.device)
        L.check(L.lib().mrep_knot_span_batch(L.ptr(dc.knots), L.ptr(dc.knot_ofs),
                                             L.ptr(dc.degree), L.ptr(cid), L.ptr(td), n,
                                             L.ptr(span), L.stream_ptr()))
        return L.to_host(span)

    def device_bytes(self):
        nb = ctypes.c_int64()
        L.check(L.lib().mrep_curveset_info(self.handle, None, None, None, ctypes.byref(nb)))
        return nb.value

    def free(self):
        if self._handle is not None:
            try:
                L.load_library().mrep_curveset_free(self._handle)
            finally:
                self._handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    CELL_MAX_BYTES = 16 << 30  # skip the index rather than spend more HBM on it

    def build_cells(self, grid_max=16, max_bytes=None):
        """Per-curve cell indices (mrep_curveset_cells_build): afterwards every
        batch scans its query's cell list instead of walking the curve's
        hierarchy -- same t / foot / dist / segment (cells are exact).  Returns
        the index size in bytes, or 0 when it would exceed max_bytes (no index)."""
        nb = ctypes.c_int64()
        rc = L.lib().mrep_curveset_cells_build(
            self.handle, int(grid_max), int(self.CELL_MAX_BYTES if max_bytes is None else max_bytes),
            ctypes.byref(nb), L.stream_ptr())
        if rc == 1 and b"budget" in L.lib().mrep_last_error():  # MREP_ERR_ARG
            return 0
        L.check(rc)
        self.cells_bytes = nb.value
        return nb.value

    # ------------------------------------------------------------ projection
    def project_device(self, queries, curve_ids, clip_tol=1e-6, max_iter=8, counters=None,
                       extra_flags=0):
        """Device tensors in, device tensors out: (t, foot, dist, cand, seg)."""
        torch = L._torch()
        q = queries if isinstance(queries, torch.Tensor) else L.to_dev(np.asarray(queries))
        cid = (curve_ids if isinstance(curve_ids, torch.Tensor)
               else L.to_dev(np.asarray(curve_ids), torch.int32))
        q = q.to(torch.float64).contiguous()
        cid = cid.to(torch.int32).contiguous()
        n = q.shape[0]
        dev = q.device
        t = torch.empty((n,), dtype=torch.float64, device=dev)
        foot = torch.empty((n, self.d), dtype=torch.float64, device=dev)
        dist = torch.empty((n,), dtype=torch.float64, device=dev)
        cand = torch.empty((n,), dtype=torch.int64, device=dev)
        seg = torch.empty((n,), dtype=torch.int32, device=dev)
        L.check(L.lib().mrep_project_batch(
            self.handle, L.ptr(q), L.ptr(cid), n, float(clip_tol), int(max_iter),
            L.MREP_SCREEN | int(extra_flags), L.ptr(t), L.ptr(foot), L.ptr(dist), L.ptr(cand),
            L.ptr(seg), L.ptr(counters), L.stream_ptr()))
        return t, foot, dist, cand, seg

    def project_host(self, queries, curve_ids, out=None, clip_tol=1e-6, max_iter=8,
                     counters=None):
        """End-to-end call on HOST arrays through mrep_project_batch_host."""
        q = np.ascontiguousarray(queries, dtype=np.float64)
        cid = np.ascontiguousarray(curve_ids, dtype=np.int32)
        n = q.shape[0]
        if out is None:
            out = (np.empty(n), np.empty((n, self.d)), np.empty(n),
                   np.empty(n, dtype=np.int64), np.empty(n, dtype=np.int32))
        t, foot, dist, cand, seg = out
        p = lambda a: ctypes.c_void_p(a.ctypes.data if a is not None else 0)  # noqa: E731
        L.check(L.lib().mrep_project_batch_host(
            self.handle, p(q), p(cid), n, float(clip_tol), int(max_iter), L.MREP_SCREEN,
            p(t), p(foot), p(dist), p(cand), p(seg),
            p(counters) if counters is not None else ctypes.c_void_p(0)))
        return out


def prepare_curve_set(curves, tolerance: float = 1e-4, batch_cap: int = 4096) -> PreparedCurveSet:
    """prepare_curve for every curve, as one batched device decomposition +
    approximation, packed into one device curve set.

    All curves must share one dimension.  Validation errors raise (use
    batched_decompose for per-curve error isolation).  batch_cap is the
    reference's per-curve cap on pending subdivisions per pass
    (reduce_approx.py:244); results never depend on it, and the device run
    uses batch_cap x len(curves) per pass.
    """
    if not tolerance > 0.0:
        raise DomainError("tolerance must be positive")
    curves = list(curves)
    if not curves:
        raise DomainError("prepare_curve_set needs at least one curve")
    dims = {c.dimension for c in curves}
    if len(dims) != 1:
        raise DomainError("all curves of a set must have the same dimension")
    for c in curves:
        validate_curve(c)
        k, p = c.knots.knots, c.degree
        if not np.any(k[p + 1: len(k) - p] > k[p: len(k) - p - 1]):  # span_indices() empty
            raise EmptyDomain("curve has no nonzero-length span")
    d = dims.pop()
    torch = L._torch()
    dcurves = DeviceCurves(curves)
    dec = decompose_device(dcurves)
    dcurves.ctrl = dcurves.ctrl_ofs = None  # knots stay for knot_spans
    cap = int(min(max(batch_cap, 1) * len(curves), 1 << 22))
    res = approximate_device(dec["rows"], dec["row_ofs"], dec["iv"], dec["curve"], dec["nseg"], d,
                             tolerance, cap)
    pts, iv, err, cid = res.fetch()
    res.free()
    counts = torch.bincount(cid.to(torch.int64), minlength=len(curves))
    ofs = np.concatenate(([0], np.cumsum(L.to_host(counts)))).astype(np.int64)
    if np.any(np.diff(ofs) < 1):
        raise GeometryError("a curve produced no cubics")
    ta = iv[:, 0].contiguous()
    tb = iv[:, 1].contiguous()
    h = ctypes.c_void_p()
    L.check(L.lib().mrep_curveset_create_dev(L.ptr(pts), L.ptr(ta), L.ptr(tb),
                                             ctypes.c_void_p(ofs.ctypes.data), len(curves), d,
                                             L.stream_ptr(), ctypes.byref(h)))
    return PreparedCurveSet(curves, tolerance, pts, ta, tb, ofs, h, err=err, dev_curves=dcurves)


def curve_set_from_prepared(preps) -> PreparedCurveSet:
    """A device curve set from already-prepared curves (e.g. reference
    PreparedCurve objects): their seg_pts / seg_ta / seg_tb are packed as is."""
    preps = list(preps)
    if not preps:
        raise DomainError("need at least one prepared curve")
    d = preps[0].seg_pts.shape[2]
    pts = np.ascontiguousarray(np.concatenate([np.asarray(p.seg_pts) for p in preps]),
                               dtype=np.float64)
    ta = np.ascontiguousarray(np.concatenate([np.asarray(p.seg_ta) for p in preps]),
                              dtype=np.float64)
    tb = np.ascontiguousarray(np.concatenate([np.asarray(p.seg_tb) for p in preps]),
                              dtype=np.float64)
    ofs = np.concatenate(([0], np.cumsum([len(p.seg_ta) for p in preps]))).astype(np.int64)
    L.lib()
    h = ctypes.c_void_p()
    p = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    L.check(L.lib().mrep_curveset_create(p(pts), p(ta), p(tb), p(ofs), len(preps), d,
                                         ctypes.byref(h)))
    curves = [getattr(pr, "curve", None) for pr in preps]
    return PreparedCurveSet(curves, getattr(preps[0], "tolerance", None), pts, ta, tb, ofs, h)


def project_batch(cset: PreparedCurveSet, queries, curve_ids, workers: int | None = None,
                  clip_tol: float = 1e-6, max_iterations: int = 8, *,
                  return_segments: bool = False, return_spans: bool = False):
    """Project query i onto curve curve_ids[i]; returns host arrays
    (t, foot, dist, cand[, seg][, span]) -- per query what
    project_prepared(cset[c], q) returns (cand: candidates the screened kernel
    examined; span: knot span of t* in curve c, core.py:108-112)."""
    if max_iterations < 1:
        raise DomainError("max_iterations must be >= 1")
    q = np.ascontiguousarray(np.atleast_2d(np.asarray(queries, dtype=np.float64)))
    if q.shape[1] != cset.d:
        raise DomainError("query dimension does not match the curve set")
    cid = np.ascontiguousarray(np.asarray(curve_ids).reshape(-1))
    if cid.shape[0] != q.shape[0]:
        raise DomainError("need one curve id per query")
    if cid.size and (cid.min() < 0 or cid.max() >= len(cset)):
        raise DomainError("curve id out of range")
    cid = cid.astype(np.int32)
    plan_work(len(q), 1 if workers is None else workers)
    n = q.shape[0]
    if n == 0:
        out = (np.empty(0), np.empty((0, cset.d)), np.empty(0), np.empty(0, np.int64))
        return (out + ((np.empty(0, np.int32),) if return_segments else ())
                + ((np.empty(0, np.int32),) if return_spans else ()))
    cnt = np.zeros(L.NUM_COUNTERS, dtype=np.uint64)
    t, foot, dist, cand, seg = cset.project_host(q, cid, clip_tol=clip_tol,
                                                 max_iter=max_iterations, counters=cnt)
    if int(cnt[L.CNT_HULL_MISS]) > 0:
        raise NoRoot("hull never crossed on a surviving piece; elimination bug")
    out = (t, foot, dist, cand)
    return (out + ((seg,) if return_segments else ())
            + ((cset.knot_spans(t, cid),) if return_spans else ()))
