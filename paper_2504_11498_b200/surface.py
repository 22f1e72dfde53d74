"""Tensor-product B-spline surfaces: decomposition into Bezier patches and
batch point projection / inversion on the B200 (BASELINE.json configs[3]).

The reference package has no surface code -- its SPEC.md:15, 98 and 497 put
surfaces out of scope -- so this module extends the curve path the way
SURVEY.md 8(c) prescribes, with the same conventions as the curve API:

* validation reuses the curve invariants (core.py:201-231) per direction;
* decompose_surface applies the reference's per-span decomposition
  (decompose.py:19-46: Q = T_p diag(h^k) A_q P, clamped ends exact) along v
  for every row of the net, then along u for every column of the row
  patches -- two batched device decompositions (mrep_decompose);
* project_surface_prepared runs the sm_100a pipeline of mrep_surface.cu:
  BVH screening over the patches, then per candidate patch the best of the
  (pu+1)(pv+1) Bernstein seeds refined by a box-constrained Newton
  iteration; the winner is the smallest distance, ties inside 1e-12 going
  to the smallest patch id (the curve path's two-pass rule, _kernels.py:
  480-490, with the patch id in place of t);
* errors: DomainError / the curve validation errors, PointNotOnCurve for a
  failed inversion (as invert_point, project.py:306-312).

Parity is pinned to the C oracle oracle/mrep_surface_oracle.c (the same
algorithm, brute force over all patches) and to a dense-grid global search.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .core import (
    BSplineCurve,
    DomainError,
    EmptyDomain,
    KnotVector,
    PointNotOnCurve,
    _freeze,
    as_readonly,
    validate_curve,
)
from .decompose import DeviceCurves, decompose_device
from .project import plan_work

SUPPORTED_DEGREES = {(1, 1), (2, 2), (3, 3), (4, 4), (5, 5), (3, 5), (5, 3)}


@dataclass(frozen=True, eq=False)
class BSplineSurface:
    """Clamped tensor-product B-spline surface with a [nu][nv][3] control net."""

    degree_u: int
    degree_v: int
    knots_u: KnotVector
    knots_v: KnotVector
    control_points: np.ndarray

    def __post_init__(self):
        if not isinstance(self.knots_u, KnotVector):
            _freeze(self, knots_u=KnotVector(self.knots_u))
        if not isinstance(self.knots_v, KnotVector):
            _freeze(self, knots_v=KnotVector(self.knots_v))
        _freeze(self, control_points=as_readonly(np.asarray(self.control_points,
                                                            dtype=np.float64)))

    @property
    def shape(self):
        return self.control_points.shape[:2]

    @property
    def domain_u(self):
        k = self.knots_u.knots
        return float(k[self.degree_u]), float(k[len(k) - self.degree_u - 1])

    @property
    def domain_v(self):
        k = self.knots_v.knots
        return float(k[self.degree_v]), float(k[len(k) - self.degree_v - 1])

    def row_curve(self, r) -> BSplineCurve:
        """Row r of the net as a curve along v."""
        return BSplineCurve(self.degree_v, self.knots_v, self.control_points[r])

    def column_curve(self, c) -> BSplineCurve:
        """Column c of the net as a curve along u."""
        return BSplineCurve(self.degree_u, self.knots_u, self.control_points[:, c])


@dataclass(frozen=True, eq=False)
class BezierPatch:
    """One polynomial patch in Bernstein form with its parameter rectangle."""

    degree_u: int
    degree_v: int
    control_points: np.ndarray  # [pu+1][pv+1][3]
    source_rect: tuple          # ((u0, u1), (v0, v1))

    def __post_init__(self):
        _freeze(self, control_points=as_readonly(self.control_points))


@dataclass(frozen=True, eq=False)
class SurfaceProjectionResult:
    query: np.ndarray
    uv: tuple
    foot: np.ndarray
    distance: float
    patch: int


def validate_surface(surface: BSplineSurface) -> BSplineSurface:
    """Curve invariants (core.py:201-231) in each direction + a 3-D net."""
    cp = surface.control_points
    if cp.ndim != 3 or cp.shape[2] != 3:
        raise DomainError(f"control net must be [nu][nv][3], got shape {cp.shape}")
    validate_curve(BSplineCurve(surface.degree_u, surface.knots_u, cp[:, 0]))
    validate_curve(BSplineCurve(surface.degree_v, surface.knots_v, cp[0]))
    return surface


def _spans(p, knots):
    return [q for q in range(p, len(knots) - p - 1) if knots[q] < knots[q + 1]]


def _decompose_device(surface):
    """Patch control points [nus][nvs][pu+1][pv+1][3] and rectangles."""
    validate_surface(surface)
    pu, pv = surface.degree_u, surface.degree_v
    ku, kv = surface.knots_u.knots, surface.knots_v.knots
    su, sv = _spans(pu, ku), _spans(pv, kv)
    if not su or not sv:
        raise EmptyDomain("surface has no nonzero-length span")
    nu, nv = surface.shape
    # pass 1: every row along v -> [nu][nvs][pv+1][3]
    rows = [surface.row_curve(r) for r in range(nu)]
    d1 = decompose_device(DeviceCurves(rows))
    R = L.to_host(d1["rows"]).reshape(nu, len(sv), pv + 1, 3)
    # pass 2: every column of the row patches along u -> [nvs][pv+1][nus][pu+1][3]
    cols = [BSplineCurve(pu, surface.knots_u, np.ascontiguousarray(R[:, j, c]))
            for j in range(len(sv)) for c in range(pv + 1)]
    d2 = decompose_device(DeviceCurves(cols))
    C = L.to_host(d2["rows"]).reshape(len(sv), pv + 1, len(su), pu + 1, 3)
    pts = np.ascontiguousarray(C.transpose(2, 0, 3, 1, 4))  # [i][j][a][c][xyz]
    iv = np.empty((len(su), len(sv), 4))
    for i, q in enumerate(su):
        iv[i, :, 0], iv[i, :, 1] = ku[q], ku[q + 1]
    for j, q in enumerate(sv):
        iv[:, j, 2], iv[:, j, 3] = kv[q], kv[q + 1]
    return pts, iv


def decompose_surface(surface: BSplineSurface) -> list[BezierPatch]:
    """One degree-(pu, pv) Bezier patch per pair of nonzero spans, row-major
    over (u-span, v-span)."""
    pts, iv = _decompose_device(surface)
    nus, nvs = pts.shape[:2]
    return [BezierPatch(surface.degree_u, surface.degree_v, pts[i, j],
                        ((iv[i, j, 0], iv[i, j, 1]), (iv[i, j, 2], iv[i, j, 3])))
            for i in range(nus) for j in range(nvs)]


class DeviceSurfaceTable:
    """Device-resident patch table + AABB hierarchy (mrep_surface_table_pack)."""

    def __init__(self, patch_pts, patch_iv, pu, pv):
        torch = L._torch()
        nus, nvs = patch_pts.shape[:2]
        self.nus, self.nvs, self.pu, self.pv = nus, nvs, pu, pv
        self.npatch = nus * nvs
        nbytes = L.lib().mrep_surface_table_bytes(self.npatch, pu, pv)
        if nbytes <= 0:
            raise DomainError("surface table needs at least one patch")
        self.buf = torch.empty((nbytes // 8,), dtype=torch.float64, device=L.device())
        P = L.to_dev(np.ascontiguousarray(patch_pts).reshape(-1))
        I = L.to_dev(np.ascontiguousarray(patch_iv).reshape(-1))
        L.check(L.lib().mrep_surface_table_pack(L.ptr(P), L.ptr(I), nus, nvs, pu, pv,
                                                L.ptr(self.buf), L.stream_ptr()))
        self.cells = None
        self.cells_tried = False
        self.use_cells = True  # False: always walk the hierarchy

    # cell index (mrep_surface_cells_build): built once, lazily, on the first
    # dense batch (queries >> patches), as for curve tables
    CELL_MIN_QUERIES = 1 << 16
    CELL_MAX_PATCHES = 1 << 17
    CELL_MAX_BYTES = 4 << 30

    def build_cells(self, grid=None):
        torch = L._torch()
        if grid is None:
            grid = 128 if self.npatch > (1 << 14) else 64
        nb = L.lib().mrep_surface_cells_bytes(L.ptr(self.buf), self.npatch, self.pu, self.pv,
                                              grid, L.stream_ptr())
        if nb <= 0:
            L.check(1)
        if nb > self.CELL_MAX_BYTES:
            return self
        try:
            self.cells = torch.empty((nb + 3) // 4, dtype=torch.int32, device=self.buf.device)
        except torch.cuda.OutOfMemoryError:
            return self  # no room: the hierarchy walk is exact without the index
        L.check(L.lib().mrep_surface_cells_build(L.ptr(self.buf), self.npatch, self.pu, self.pv,
                                                  grid, L.ptr(self.cells), nb, L.stream_ptr()))
        return self

    def _cell_flag(self, n):
        if not self.use_cells or self.npatch > self.CELL_MAX_PATCHES:
            return 0
        if (self.cells is None and not self.cells_tried
                and n >= max(self.CELL_MIN_QUERIES, 8 * self.npatch)):
            self.cells_tried = True
            self.build_cells()
        return L.MREP_CELLS if (self.cells is not None and n >= 8 * self.npatch) else 0

    def project(self, queries, counters=None, extra_flags=0):
        """Device queries (n, 3) -> device (u, v, foot, dist, patch)."""
        torch = L._torch()
        q = queries if isinstance(queries, torch.Tensor) else L.to_dev(np.asarray(queries))
        q = q.to(torch.float64).contiguous()
        n = q.shape[0]
        dev = q.device
        u = torch.empty((n,), dtype=torch.float64, device=dev)
        v = torch.empty((n,), dtype=torch.float64, device=dev)
        foot = torch.empty((n, 3), dtype=torch.float64, device=dev)
        dist = torch.empty((n,), dtype=torch.float64, device=dev)
        patch = torch.empty((n,), dtype=torch.int32, device=dev)
        L.check(L.lib().mrep_project_surface(
            L.ptr(self.buf), self.npatch, self.pu, self.pv, L.ptr(q), n,
            int(extra_flags) | self._cell_flag(n), L.ptr(u), L.ptr(v), L.ptr(foot), L.ptr(dist), L.ptr(patch), L.ptr(counters),
            L.stream_ptr()))
        return u, v, foot, dist, patch

    def project_host(self, queries, out=None, counters=None, extra_flags=0):
        q = np.ascontiguousarray(queries, dtype=np.float64)
        n = q.shape[0]
        if out is None:
            out = (np.empty(n), np.empty(n), np.empty((n, 3)), np.empty(n),
                   np.empty(n, dtype=np.int32))
        u, v, foot, dist, patch = out
        p = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
        L.check(L.lib().mrep_project_surface_host(
            L.ptr(self.buf), self.npatch, self.pu, self.pv, p(q), n,
            int(extra_flags) | self._cell_flag(n), p(u),
            p(v), p(foot), p(dist), p(patch),
            p(counters) if counters is not None else ctypes.c_void_p(0)))
        return out


class PreparedSurface:
    """Bezier patches of a surface (host, read-only) + the device table."""

    def __init__(self, surface, patch_pts, patch_iv):
        self.surface = surface
        self.patch_pts = as_readonly(patch_pts)  # [nus][nvs][pu+1][pv+1][3]
        self.patch_iv = as_readonly(patch_iv)    # [nus][nvs][4]
        self._table = None

    @property
    def num_patches(self):
        return self.patch_pts.shape[0] * self.patch_pts.shape[1]

    @property
    def table(self) -> DeviceSurfaceTable:
        if self._table is None:
            self._table = DeviceSurfaceTable(self.patch_pts, self.patch_iv,
                                             self.surface.degree_u, self.surface.degree_v)
        return self._table


def prepare_surface(surface: BSplineSurface) -> PreparedSurface:
    """Decompose on the GPU and keep the patch table resident."""
    if (surface.degree_u, surface.degree_v) not in SUPPORTED_DEGREES:
        raise DomainError(f"surface degrees {(surface.degree_u, surface.degree_v)} not in "
                          f"{sorted(SUPPORTED_DEGREES)}")
    pts, iv = _decompose_device(surface)
    prep = PreparedSurface(surface, pts, iv)
    prep.table  # noqa: B018  (build the device table now)
    return prep


def project_surface_prepared(prep: PreparedSurface, queries, workers: int | None = None, *,
                             return_patches: bool = False):
    """(u, v, foot, dist[, patch]) host arrays for every 3-D query."""
    q = np.ascontiguousarray(np.atleast_2d(np.asarray(queries, dtype=np.float64)))
    if q.shape[1] != 3:
        raise DomainError("surface queries must be 3-D")
    plan_work(len(q), 1 if workers is None else workers)
    if len(q) == 0:
        out = (np.empty(0), np.empty(0), np.empty((0, 3)), np.empty(0))
        return out + ((np.empty(0, np.int32),) if return_patches else ())
    u, v, foot, dist, patch = prep.table.project_host(q)
    out = (u, v, foot, dist)
    return out + ((patch,) if return_patches else ())


def project_surface_points(surface: BSplineSurface, queries,
                           workers: int | None = None) -> list[SurfaceProjectionResult]:
    prep = prepare_surface(surface)
    q = np.atleast_2d(np.asarray(queries, dtype=np.float64))
    u, v, foot, dist, patch = project_surface_prepared(prep, q, workers, return_patches=True)
    return [SurfaceProjectionResult(q[i], (float(u[i]), float(v[i])), foot[i], float(dist[i]),
                                    int(patch[i])) for i in range(len(q))]


def invert_surface_point(surface: BSplineSurface, q, tolerance: float = 1e-4):
    """(u, v) of a point on the surface; PointNotOnCurve beyond 10 * tolerance."""
    if not tolerance > 0.0:
        raise DomainError("tolerance must be positive")
    r = project_surface_points(surface, [q])[0]
    if r.distance > 10.0 * tolerance:
        raise PointNotOnCurve(f"projection distance {r.distance:.3e} exceeds 10 * {tolerance}")
    return r.uv


def eval_surface(surface: BSplineSurface, uv) -> np.ndarray:
    """Surface points at parameter pairs uv [n][2] (tensor Cox-de Boor, GPU)."""
    uv = np.ascontiguousarray(np.atleast_2d(np.asarray(uv, dtype=np.float64)))
    (u0, u1), (v0, v1) = surface.domain_u, surface.domain_v
    if np.any(uv[:, 0] < u0) or np.any(uv[:, 0] > u1) or np.any(uv[:, 1] < v0) \
            or np.any(uv[:, 1] > v1):
        raise DomainError("parameter outside the surface domain")
    nu, nv = surface.shape
    ku, kv = L.to_dev(surface.knots_u.knots), L.to_dev(surface.knots_v.knots)
    cp = L.to_dev(np.ascontiguousarray(surface.control_points).reshape(-1))
    uvd = L.to_dev(uv)
    out = L.empty((len(uv), 3))
    if len(uv):
        L.check(L.lib().mrep_eval_surface(surface.degree_u, surface.degree_v, L.ptr(ku),
                                          len(surface.knots_u.knots), L.ptr(kv),
                                          len(surface.knots_v.knots), L.ptr(cp), nu, nv,
                                          L.ptr(uvd), len(uv), L.ptr(out), L.stream_ptr()))
    return L.to_host(out)
