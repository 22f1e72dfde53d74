"""Nearest-over-set projection: every query is
projected onto the NEAREST of many prepared curves.

The reference has no such call (SPEC.md:497 lists it as a non-goal); a user
would call project_prepared (project.py:245-289) once per curve and keep the
minimum.  Here the cubics of all curves go into ONE segment table, so one
screened projection (the same wavefront kernels, AABB hierarchy and cell
index as a single curve) culls across curves.  Between two curves sits a
separator record (NaN interval, empty box): it is never tested in range, and
its two seams are the previous curve's end point and the next curve's start
point, so every curve keeps exactly its own seams and cubics.

Per query the result is the candidate of minimum distance over all curves;
within 1e-12 of that minimum the reference's tie rule applies to the merged
candidate set (smallest parameter t, then the smallest global cubic/seam
order).  Distances equal the minimum of the per-curve project_prepared
distances bit for bit (tests/test_gpu_nearest.py).
"""

import numpy as np

from . import _device as D
from . import _lib as L
from .core import DomainError
from .project import PreparedCurve


class PreparedNearestSet:
    """Prepared curves merged into one device segment table."""

    def __init__(self, preps):
        preps = list(preps)
        if not preps:
            raise DomainError("a nearest-over-set table needs at least one curve")
        d = preps[0].seg_pts.shape[2]
        if any(p.seg_pts.shape[2] != d for p in preps):
            raise DomainError("all curves of a set must have the same dimension")
        self.preps = preps
        self.d = d
        self.counts = np.array([len(p.seg_ta) for p in preps], dtype=np.int64)
        # global index of each curve's first cubic (one separator between curves)
        self.starts = np.concatenate(([0], np.cumsum(self.counts + 1)[:-1])).astype(np.int64)
        pts, ta, tb, st, sp = [], [], [], [], []
        sep_pts = np.full((1, 4, d), np.nan)
        for i, p in enumerate(preps):
            if i:
                pts.append(sep_pts)
                ta.append([np.nan])
                tb.append([np.nan])
            pts.append(p.seg_pts)
            ta.append(p.seg_ta)
            tb.append(p.seg_tb)
            st.append(p.seam_t)
            sp.append(p.seam_pt)
        self.table = D.DeviceTable(np.concatenate(pts), np.concatenate(ta), np.concatenate(tb),
                                   np.concatenate(st), np.concatenate(sp))
        self.S = self.table.S

    def locate(self, seg):
        """Global winning index -> (curve id, cubic index within the curve).
        A seam candidate at a curve's start point reports the separator
        before it; it belongs to that curve's cubic 0 (the reference's seam-0
        convention)."""
        seg = np.asarray(seg, dtype=np.int64)
        cid = np.searchsorted(self.starts, seg, side="right") - 1
        local = seg - self.starts[cid]
        at_sep = local >= self.counts[cid]
        cid = np.where(at_sep, cid + 1, cid)
        local = np.where(at_sep, 0, local)
        return cid.astype(np.int32), local.astype(np.int32)


def prepare_nearest_set(preps) -> PreparedNearestSet:
    """Merge prepared curves (PreparedCurve, same dimension) into one table."""
    for p in preps:
        if not isinstance(p, PreparedCurve):
            raise DomainError("prepare_nearest_set takes PreparedCurve objects")
    return PreparedNearestSet(preps)


def project_nearest(nset: PreparedNearestSet, queries, clip_tol: float = 1e-6,
                    max_iterations: int = 8):
    """(curve_id, t, foot, distance, segment) per query: the nearest curve of
    the set, the parameter and foot point on it, and the winning cubic's
    index within that curve."""
    q = np.ascontiguousarray(np.atleast_2d(np.asarray(queries, dtype=np.float64)))
    if q.ndim != 2 or q.shape[1] != nset.d:
        raise DomainError(f"queries must be (n, {nset.d})")
    if max_iterations < 1:
        raise DomainError("max_iterations must be >= 1")
    n = q.shape[0]
    if n == 0:
        return (np.empty(0, np.int32), np.empty(0), np.empty((0, nset.d)), np.empty(0),
                np.empty(0, np.int32))
    # per-query walks offer both seams of every visited cubic (the group
    # walk offers end seams only, which needs the previous cubic's box to
    # hold the start seam -- not true after a separator)
    tab = nset.table
    mode = 0 if n >= 8 * tab.S else L.MREP_PER_LANE
    t, foot, dist, _, seg = tab.project_host(q, clip_tol=clip_tol, max_iter=max_iterations,
                                             screen=True, extra_flags=mode)
    cid, local = nset.locate(seg)
    return cid, t, foot, dist, local
