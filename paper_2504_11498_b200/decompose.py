"""B-spline -> piecewise Bezier on the GPU -- the reference's decompose.py surface.

decompose_to_bezier / batched_decompose (decompose.py:19-67) run as ONE
batched launch over all curves: a per-curve span count + exclusive scan
(mrep_decompose_plan), then one warp per nonzero span computing
Q = T_p diag(h^k) A_q P (mrep_decompose).  Validation stays on the host, and a
curve that fails it is reported in place by batched_decompose, as in the
reference.
"""

import numpy as np

from . import _lib as L
from .core import BezierSegment, BSplineCurve, EmptyDomain, GeometryError, validate_curve


class DeviceCurves:
    """CSR device copy of a list of validated curves (all of one dimension)."""

    def __init__(self, curves):
        torch = L._torch()
        self.curves = list(curves)
        self.d = self.curves[0].dimension
        deg = np.array([c.degree for c in self.curves], dtype=np.int32)
        kl = [len(c.knots.knots) for c in self.curves]
        cl = [c.control_points.shape[0] for c in self.curves]
        self.knot_ofs_h = np.concatenate(([0], np.cumsum(kl))).astype(np.int64)
        self.ctrl_ofs_h = np.concatenate(([0], np.cumsum(cl))).astype(np.int64)
        self.degree = L.to_dev(deg, torch.int32)
        self.knot_ofs = L.to_dev(self.knot_ofs_h, torch.int64)
        self.ctrl_ofs = L.to_dev(self.ctrl_ofs_h, torch.int64)
        self.knots = L.to_dev(np.concatenate([c.knots.knots for c in self.curves]))
        self.ctrl = L.to_dev(np.concatenate([c.control_points for c in self.curves]))
        self.nc = len(self.curves)


def decompose_device(dc: DeviceCurves):
    """Run the batched decomposition; returns a dict of device tensors.

    rows [R][d], row_ofs [S+1], iv [S][2], curve [S], span [S], seg_ofs [nc+1].
    """
    torch = L._torch()
    lib = L.lib()
    seg_ofs = L.empty((dc.nc + 1,), torch.int64)
    row_base = L.empty((dc.nc + 1,), torch.int64)
    import ctypes
    ns = ctypes.c_int64()
    nr = ctypes.c_int64()
    L.check(lib.mrep_decompose_plan(L.ptr(dc.degree), L.ptr(dc.knot_ofs), L.ptr(dc.knots), dc.nc,
                                    L.ptr(seg_ofs), L.ptr(row_base), ctypes.byref(ns),
                                    ctypes.byref(nr), L.stream_ptr()))
    S, R = ns.value, nr.value
    out = dict(seg_ofs=seg_ofs, nseg=S, d=dc.d)
    if S == 0:
        return out
    out["rows"] = L.empty((R, dc.d))
    out["row_ofs"] = L.empty((S + 1,), torch.int64)
    out["iv"] = L.empty((S, 2))
    out["curve"] = L.empty((S,), torch.int32)
    out["span"] = L.empty((S,), torch.int32)
    L.check(lib.mrep_decompose(L.ptr(dc.degree), L.ptr(dc.knot_ofs), L.ptr(dc.knots),
                               L.ptr(dc.ctrl_ofs), L.ptr(dc.ctrl), dc.nc, dc.d, L.ptr(seg_ofs),
                               L.ptr(row_base), S, L.ptr(out["rows"]), L.ptr(out["row_ofs"]),
                               L.ptr(out["iv"]), L.ptr(out["curve"]), L.ptr(out["span"]),
                               L.stream_ptr()))
    return out


def _segments_from(dec, curves):
    """Host BezierSegment lists per curve from a device decomposition."""
    if dec["nseg"] == 0:
        return [[] for _ in curves]
    rows = L.to_host(dec["rows"])
    row_ofs = L.to_host(dec["row_ofs"])
    iv = L.to_host(dec["iv"])
    seg_ofs = L.to_host(dec["seg_ofs"])
    out = []
    for c, curve in enumerate(curves):
        segs = []
        for s in range(seg_ofs[c], seg_ofs[c + 1]):
            segs.append(BezierSegment(curve.degree, rows[row_ofs[s]: row_ofs[s + 1]],
                                      (iv[s, 0], iv[s, 1])))
        out.append(segs)
    return out


def decompose_to_bezier(curve: BSplineCurve) -> list[BezierSegment]:
    """One degree-p Bezier segment per nonzero-length span, in parameter order."""
    validate_curve(curve)
    if not curve.span_indices():
        raise EmptyDomain("curve has no nonzero-length span")
    dec = decompose_device(DeviceCurves([curve]))
    return _segments_from(dec, [curve])[0]


def batched_decompose(curves, workers: int | None = None):
    """Decompose many curves in one device launch; failures reported in place.

    `workers` is accepted for API compatibility (the device batch needs no
    thread pool); output order never depends on it.
    """
    curves = list(curves)
    result = [None] * len(curves)
    ok = {2: [], 3: []}
    for i, c in enumerate(curves):
        try:
            validate_curve(c)
            if not c.span_indices():
                raise EmptyDomain("curve has no nonzero-length span")
            ok[c.dimension].append(i)
        except GeometryError as exc:
            result[i] = exc
    for d, idx in ok.items():
        if not idx:
            continue
        batch = [curves[i] for i in idx]
        segs = _segments_from(decompose_device(DeviceCurves(batch)), batch)
        for i, s in zip(idx, segs):
            result[i] = s
    return result
