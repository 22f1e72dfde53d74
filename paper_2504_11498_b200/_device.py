"""Batched device operations over libmrep (numpy in, numpy out).

Each function moves its inputs to the GPU, runs one libmrep kernel and
returns host arrays.  They back the public single-pair ops of the reference
(project.py:124-209, distance.py:34-94) and the parity tests; the batch
projection itself keeps its data on the device (see project.py).
"""

import os

import numpy as np

from . import _lib as L


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def quartic_roots(coeffs):
    """_kernels._quartic_block: (n,5) -> roots (n,4) (NaN-padded), counts (n,)."""
    torch = L._torch()
    c = L.to_dev(_f64(coeffs).reshape(-1, 5))
    n = c.shape[0]
    roots = torch.full((n, 4), float("nan"), dtype=torch.float64, device=c.device)
    counts = L.empty((n,), torch.int64)
    L.check(L.lib().mrep_quartic_roots(L.ptr(c), n, L.ptr(roots), L.ptr(counts), L.stream_ptr()))
    return L.to_host(roots), L.to_host(counts)


def newton_quartic_roots(coeffs):
    """_kernels._newton_quartic_block (the bench's multistart-Newton baseline)."""
    torch = L._torch()
    c = L.to_dev(_f64(coeffs).reshape(-1, 5))
    n = c.shape[0]
    roots = torch.full((n, 4), float("nan"), dtype=torch.float64, device=c.device)
    counts = L.empty((n,), torch.int64)
    L.check(L.lib().mrep_newton_quartic_roots(L.ptr(c), n, L.ptr(roots), L.ptr(counts),
                                              L.stream_ptr()))
    return L.to_host(roots), L.to_host(counts)


def distance_poly(P, q):
    """_kernels._distance_poly batched: P (n,4,d), q (n,d) -> e (n,6)."""
    P = _f64(P)
    q = _f64(q)
    if P.ndim == 2:
        P = P[None]
        q = q[None]
    n, _, d = P.shape
    Pd, qd = L.to_dev(P), L.to_dev(q)
    e = L.empty((n, 6))
    L.check(L.lib().mrep_distance_poly(L.ptr(Pd), L.ptr(qd), n, d, L.ptr(e), L.stream_ptr()))
    return L.to_host(e)


def restrict_ordinates(b, lo, hi):
    b = _f64(b).reshape(-1, 6)
    n = b.shape[0]
    lo = np.broadcast_to(_f64(lo), (n,)).copy()
    hi = np.broadcast_to(_f64(hi), (n,)).copy()
    bd, lod, hid = L.to_dev(b), L.to_dev(lo), L.to_dev(hi)
    out = L.empty((n, 6))
    L.check(L.lib().mrep_restrict_ordinates(L.ptr(bd), L.ptr(lod), L.ptr(hid), n, L.ptr(out),
                                            L.stream_ptr()))
    return L.to_host(out)


def eval_ordinates(b, u):
    b = _f64(b).reshape(-1, 6)
    n = b.shape[0]
    u = np.broadcast_to(_f64(u), (n,)).copy()
    bd, ud = L.to_dev(b), L.to_dev(u)
    out = L.empty((n,))
    L.check(L.lib().mrep_eval_ordinates(L.ptr(bd), L.ptr(ud), n, L.ptr(out), L.stream_ptr()))
    return L.to_host(out)


def hull_cross(b):
    torch = L._torch()
    b = _f64(b).reshape(-1, 6)
    n = b.shape[0]
    bd = L.to_dev(b)
    found = L.empty((n,), torch.int32)
    z = L.empty((n, 2))
    L.check(L.lib().mrep_hull_cross(L.ptr(bd), n, L.ptr(found), L.ptr(z), L.stream_ptr()))
    return L.to_host(found).astype(bool), L.to_host(z)


def clip_root(b, tol, max_iter):
    torch = L._torch()
    b = _f64(b).reshape(-1, 6)
    n = b.shape[0]
    bd = L.to_dev(b)
    root = L.empty((n,))
    ok = L.empty((n,), torch.int32)
    used = L.empty((n,), torch.int32)
    widths = L.empty((n, max(int(max_iter), 1)))
    L.check(L.lib().mrep_clip_root(L.ptr(bd), n, float(tol), int(max_iter), L.ptr(root),
                                   L.ptr(ok), L.ptr(used), L.ptr(widths), L.stream_ptr()))
    return (L.to_host(root), L.to_host(ok).astype(bool), L.to_host(used),
            L.to_host(widths)[:, : int(max_iter)])


def ordinates_op(op, b, a=None, c=None, tol=1e-6, max_iter=8):
    """Any-degree scalar Bernstein op (mrep_ordinates_op) on rows b (n, deg+1):
    op 0 eval at a -> (n,); 1 hull -> (found (n,), z (n, 2)); 2 restrict to
    [a, c] -> (n, deg+1); 3 clip_root -> (root, ok, used, widths)."""
    torch = L._torch()
    b = _f64(b)
    b = b.reshape(-1, b.shape[-1])
    n, deg = b.shape[0], b.shape[1] - 1
    bd = L.to_dev(b)
    ad = L.to_dev(np.broadcast_to(_f64(a), (n,)).copy()) if a is not None else None
    cd = L.to_dev(np.broadcast_to(_f64(c), (n,)).copy()) if c is not None else None
    shape = {0: (n,), 1: (n, 2), 2: (n, deg + 1), 3: (n,)}[op]
    out = L.empty(shape)
    i0 = L.empty((n,), torch.int32)
    i1 = L.empty((n,), torch.int32)
    widths = L.empty((n, max(int(max_iter), 1))) if op == 3 else None
    L.check(L.lib().mrep_ordinates_op(int(op), L.ptr(bd), deg, n, L.ptr(ad), L.ptr(cd),
                                      float(tol), int(max_iter), L.ptr(out), L.ptr(i0),
                                      L.ptr(i1), L.ptr(widths), L.stream_ptr()))
    if op == 1:
        return L.to_host(i0).astype(bool), L.to_host(out)
    if op == 3:
        return (L.to_host(out), L.to_host(i0).astype(bool), L.to_host(i1),
                L.to_host(widths)[:, : int(max_iter)])
    return L.to_host(out)


def cubic_points(P, u):
    P = _f64(P)
    if P.ndim == 2:
        P = P[None]
    n, _, d = P.shape
    u = np.broadcast_to(_f64(u), (n,)).copy()
    Pd, ud = L.to_dev(P), L.to_dev(u)
    out = L.empty((n, d))
    L.check(L.lib().mrep_cubic_points(L.ptr(Pd), L.ptr(ud), n, d, L.ptr(out), L.stream_ptr()))
    return L.to_host(out)


def rebase(e):
    e = _f64(e).reshape(-1, 6)
    n = e.shape[0]
    ed = L.to_dev(e)
    out = L.empty((n, 6))
    L.check(L.lib().mrep_rebase(L.ptr(ed), n, L.ptr(out), L.stream_ptr()))
    return L.to_host(out)


def project_block(seg_pts, seg_ta, seg_tb, seam_t, seam_pt, queries, clip_tol=1e-6,
                  max_iter=8, soundness_samples=0):
    """Drop-in for _kernels._project_block on host arrays (brute force + stats)."""
    torch = L._torch()
    sp, ta, tb = L.to_dev(_f64(seg_pts)), L.to_dev(_f64(seg_ta)), L.to_dev(_f64(seg_tb))
    st, spt = L.to_dev(_f64(seam_t)), L.to_dev(_f64(seam_pt))
    q = L.to_dev(_f64(np.atleast_2d(queries)))
    S, _, d = sp.shape
    n = q.shape[0]
    out_t, out_foot, out_dist = L.empty((n,)), L.empty((n, d)), L.empty((n,))
    out_cand = L.empty((n,), torch.int64)
    out_stats = torch.zeros((n, 6), dtype=torch.int64, device=q.device)
    out_sound = L.empty((n,))
    L.check(L.lib().mrep_project_block(
        L.ptr(sp), L.ptr(ta), L.ptr(tb), L.ptr(st), L.ptr(spt), S, d, L.ptr(q), n,
        float(clip_tol), int(max_iter), int(soundness_samples), L.ptr(out_t), L.ptr(out_foot),
        L.ptr(out_dist), L.ptr(out_cand), L.ptr(out_stats), L.ptr(out_sound), L.stream_ptr()))
    return (L.to_host(out_t), L.to_host(out_foot), L.to_host(out_dist), L.to_host(out_cand),
            L.to_host(out_stats), L.to_host(out_sound))


class DeviceTable:
    """Device-resident segment table of one prepared curve (+ its AABB tree).

    Built once from the packed arrays of a PreparedCurve (project.py:225-238)
    by ``mrep_table_pack``; reused by every projection batch.
    """

    def __init__(self, seg_pts, seg_ta, seg_tb, seam_t, seam_pt):
        torch = L._torch()
        sp = seg_pts if isinstance(seg_pts, torch.Tensor) else L.to_dev(_f64(seg_pts))
        self.S, _, self.d = sp.shape
        args = [x if isinstance(x, torch.Tensor) else L.to_dev(_f64(x))
                for x in (seg_ta, seg_tb, seam_t, seam_pt)]
        nbytes = L.lib().mrep_table_bytes(self.S)
        if nbytes <= 0:
            raise ValueError("segment table needs at least one cubic")
        self.buf = torch.empty((nbytes // 8,), dtype=torch.float64, device=sp.device)
        L.check(L.lib().mrep_table_pack(L.ptr(sp), *[L.ptr(a) for a in args], self.S, self.d,
                                        L.ptr(self.buf), L.stream_ptr()))
        self.cells = None
        self.cells_tried = False
        self.cand_cells = None
        self.cand_tried = False

    # a cell index pays off for dense batches (queries >> cubics); built once,
    # lazily, on the first such batch (mrep_cells_build)
    CELL_MIN_QUERIES = 1 << 16
    CELL_MAX_CUBICS = 1 << 17
    CELL_MAX_BYTES = 16 << 30  # skip the index rather than spend more HBM on it

    def build_cells(self, grid=None):
        torch = L._torch()
        if grid is None and os.environ.get("MREP_CELL_GRID"):  # A/B override
            grid = int(os.environ["MREP_CELL_GRID"])
        if grid is None:
            big = self.S > (1 << 14)
            # big tables: 256^3; from 2^16 cubics 384^3 (cfg5, 10^5 cubics:
            # 11.7 GB built in 4.2 s, projection 8% faster than 256^3 with
            # 5.7 GB / 2.0 s; cfg6's 41k cubics gain 1% for 3x the build)
            huge = self.S >= (1 << 16)
            grid = ((384 if huge else 256) if big else 64) if self.d == 3 else (512 if big else 256)
        nb = L.lib().mrep_cells_bytes(L.ptr(self.buf), self.S, self.d, grid, L.stream_ptr())
        if nb <= 0:
            L.check(1)
        if nb > self.CELL_MAX_BYTES:
            return self
        try:
            self.cells = torch.empty((nb + 3) // 4, dtype=torch.int32, device=self.buf.device)
        except torch.cuda.OutOfMemoryError:
            return self  # no room: the hierarchy walk is exact without the index
        L.check(L.lib().mrep_cells_build(L.ptr(self.buf), self.S, self.d, grid,
                                          L.ptr(self.cells), nb, L.stream_ptr()))
        return self

    def _cell_flag(self, n, screen):
        if not screen or self.S > self.CELL_MAX_CUBICS:
            return 0
        if self.cells is None and not self.cells_tried and n >= max(self.CELL_MIN_QUERIES,
                                                                    8 * self.S):
            self.cells_tried = True
            self.build_cells()
        return L.MREP_CELLS if (self.cells is not None and n >= 8 * self.S) else 0

    # the exact-cand pass (MREP_CAND_EXACT) tests every (query, cubic) pair
    # unless the table has a cand cell index; built lazily once the pass is
    # large enough to pay for it (mrep_cand_cells_build: cfg2 ~5 ms, 19 MB)
    CAND_MIN_PAIRS = 1 << 24
    CAND_MAX_BYTES = 4 << 30

    def build_cand_cells(self, grid=None):
        torch = L._torch()
        if grid is None:
            grid = 32 if self.d == 3 else 128
        nb = L.lib().mrep_cand_cells_bytes(L.ptr(self.buf), self.S, self.d, grid, L.stream_ptr())
        if nb <= 0:
            L.check(1)
        if nb > self.CAND_MAX_BYTES:
            return self
        try:
            buf = torch.empty((nb + 3) // 4, dtype=torch.int32, device=self.buf.device)
        except torch.cuda.OutOfMemoryError:
            return self  # the full pass is exact without the index
        L.check(L.lib().mrep_cand_cells_build(L.ptr(self.buf), self.S, self.d, grid,
                                               L.ptr(buf), nb, L.stream_ptr()))
        self.cand_cells = buf
        return self

    def _cand_flag(self, n, flags):
        if not (flags & L.MREP_CAND_EXACT) or (flags & L.MREP_CAND_CELLS):
            return 0
        if self.cand_cells is None and not self.cand_tried and n * self.S >= self.CAND_MIN_PAIRS:
            self.cand_tried = True
            self.build_cand_cells()
        return L.MREP_CAND_CELLS if self.cand_cells is not None else 0

    def project(self, queries, clip_tol=1e-6, max_iter=8, soundness_samples=0, screen=True,
                stats=False, counters=None, extra_flags=0):
        """Project device queries (n, d); returns device tensors
        (t, foot, dist, cand, seg, stats|None, sound|None)."""
        torch = L._torch()
        q = queries if isinstance(queries, torch.Tensor) else L.to_dev(_f64(queries))
        q = q.contiguous()
        n = q.shape[0]
        dev = q.device
        t = torch.empty((n,), dtype=torch.float64, device=dev)
        foot = torch.empty((n, self.d), dtype=torch.float64, device=dev)
        dist = torch.empty((n,), dtype=torch.float64, device=dev)
        cand = torch.empty((n,), dtype=torch.int64, device=dev)
        seg = torch.empty((n,), dtype=torch.int32, device=dev)
        st = torch.zeros((n, 6), dtype=torch.int64, device=dev) if stats else None
        sound = torch.empty((n,), dtype=torch.float64, device=dev) if stats else None
        flags = (L.MREP_STATS if stats else 0) | (L.MREP_SCREEN if (screen and not stats) else 0)
        flags |= int(extra_flags)
        if not (extra_flags & (L.MREP_PACKET | L.MREP_PER_LANE | L.MREP_GROUP)):
            flags |= self._cell_flag(n, screen and not stats)
        flags |= self._cand_flag(n, flags)
        L.check(L.lib().mrep_project(
            L.ptr(self.buf), self.S, self.d, L.ptr(q), n, float(clip_tol), int(max_iter),
            int(soundness_samples), flags, L.ptr(t), L.ptr(foot), L.ptr(dist), L.ptr(cand),
            L.ptr(seg), L.ptr(st), L.ptr(sound), L.ptr(counters), L.stream_ptr()))
        return t, foot, dist, cand, seg, st, sound

    def project_host(self, queries, out=None, clip_tol=1e-6, max_iter=8, screen=True,
                     counters=None, extra_flags=0):
        """End-to-end call on HOST arrays through mrep_project_host."""
        q = np.ascontiguousarray(queries, dtype=np.float64)
        n = q.shape[0]
        if out is None:
            out = (np.empty(n), np.empty((n, self.d)), np.empty(n),
                   np.empty(n, dtype=np.int64), np.empty(n, dtype=np.int32))
        t, foot, dist, cand, seg = out
        import ctypes
        p = lambda a: ctypes.c_void_p(a.ctypes.data if a is not None else 0)  # noqa: E731
        flags = (L.MREP_SCREEN | self._cell_flag(n, True)) if screen else 0
        flags |= int(extra_flags)
        flags |= self._cand_flag(n, flags)
        L.check(L.lib().mrep_project_host(
            L.ptr(self.buf), self.S, self.d, p(q), n, float(clip_tol), int(max_iter),
            flags, p(t), p(foot), p(dist), p(cand), p(seg),
            p(counters) if counters is not None else ctypes.c_void_p(0)))
        return out
