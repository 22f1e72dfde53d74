"""CPU ORACLE (test infrastructure): numpy restatement of the reference's
per-curve preprocessing, i.e. everything `prepare_curve` (project.py:220-242)
runs before the projection kernel:

* constant matrices  -- basis.py:17-22 (Pascal), 76-92 (T_n), 95-107 (Gram),
  172-189 (subdivision), 192-196 (Bernstein design)
* span decomposition -- basis.py:110-149 (symbolic Cox-de Boor per span),
  decompose.py:19-46 (Q = T_p diag(h^k) A P, exact clamped ends)
* cubic approximation -- reduce_approx.py:60-121 (G1 reduction), 129-143
  (elevation), 146-155 (max error on a uniform grid), 171-182 (restriction),
  207-301 (level loop with argmax splitting and C0 snapping)

Curves are passed as plain (degree, knots, ctrl) arrays; segments as
(points, (ta, tb)).  The numpy expressions mirror the reference's, so on the
same BLAS the output matches it bit for bit (pinned in
tests/test_oracle_pin.py against tests/golden/prep.npz).  Only tests and
bench.py's CPU baseline may import this module.
"""

import numpy as np

_ROWS = 64
_PASCAL = np.zeros((_ROWS, _ROWS))
_PASCAL[:, 0] = 1.0
for _r in range(1, _ROWS):
    _PASCAL[_r, 1: _r + 1] = _PASCAL[_r - 1, : _r] + _PASCAL[_r - 1, 1: _r + 1]


def C(n, k):
    return _PASCAL[n, k] if 0 <= k <= n else 0.0


_T, _G = {}, {}


def T(n):
    """power -> Bernstein: T[i, j] = C(i, j) / C(n, j), j <= i."""
    if n not in _T:
        M = np.zeros((n + 1, n + 1))
        for i in range(n + 1):
            for j in range(i + 1):
                M[i, j] = C(i, j) / C(n, j)
        _T[n] = M
    return _T[n]


def gram(m, n):
    """integral of B_{i,m} B_{j,n} over [0, 1]."""
    if (m, n) not in _G:
        M = np.empty((m + 1, n + 1))
        for i in range(m + 1):
            for j in range(n + 1):
                M[i, j] = C(m, i) * C(n, j) / ((m + n + 1) * C(m + n, i + j))
        _G[(m, n)] = M
    return _G[(m, n)]


def split_matrices(z, n=3):
    SL = np.zeros((n + 1, n + 1))
    SR = np.zeros((n + 1, n + 1))
    for i in range(n + 1):
        for j in range(i + 1):
            SL[i, j] = C(i, j) * z ** j * (1.0 - z) ** (i - j)
    for i in range(n + 1):
        for j in range(i, n + 1):
            SR[i, j] = C(n - i, j - i) * z ** (j - i) * (1.0 - z) ** (n - j)
    return SL, SR


def design(n, us):
    us = np.asarray(us, dtype=np.float64)
    return np.stack([C(n, j) * us ** j * (1.0 - us) ** (n - j) for j in range(n + 1)], axis=1)


def de_casteljau(points, u):
    """Points of a Bezier at scalar u (core.py:248-258 for one parameter)."""
    b = np.array(points, dtype=np.float64)[None]
    uu = np.asarray(u, dtype=np.float64).reshape(-1, 1, 1)
    for _ in range(b.shape[1] - 1):
        b = (1.0 - uu) * b[:, :-1, :] + uu * b[:, 1:, :]
    return b[0, 0, :]


# ------------------------------------------------------------- decomposition
def span_basis(knots, p, q, center):
    """Coefficients (powers of t - center) of N_{q-p+j,p} on span q, column j."""
    level = {q: np.concatenate(([1.0], np.zeros(p)))}
    for j in range(1, p + 1):
        nxt = {}
        for i in range(q - j, q + 1):
            c = np.zeros(p + 1)
            a = level.get(i)
            if a is not None:
                den = knots[i + j] - knots[i]
                c[1:] += a[:-1] / den
                c += (center - knots[i]) / den * a
            b = level.get(i + 1)
            if b is not None:
                den = knots[i + j + 1] - knots[i + 1]
                c[1:] -= b[:-1] / den
                c += (knots[i + j + 1] - center) / den * b
            nxt[i] = c
        level = nxt
    return np.stack([level[q - p + j] for j in range(p + 1)], axis=1)


def nonzero_spans(p, knots):
    return [q for q in range(p, len(knots) - p - 1) if knots[q] < knots[q + 1]]


def decompose(p, knots, ctrl):
    """One degree-p Bezier (points, (ta, tb)) per nonzero span."""
    knots = np.asarray(knots, dtype=np.float64)
    ctrl = np.asarray(ctrl, dtype=np.float64)
    Tp = T(p)
    spans = nonzero_spans(p, knots)
    out = []
    for q in spans:
        h = knots[q + 1] - knots[q]
        A = span_basis(knots, p, q, knots[q])
        Q = Tp @ ((h ** np.arange(p + 1))[:, None] * A @ ctrl[q - p: q + 1])
        if q == spans[0]:
            Q[0] = ctrl[0]
        if q == spans[-1]:
            Q[p] = ctrl[-1]
        out.append((Q, (float(knots[q]), float(knots[q + 1]))))
    return out


# ------------------------------------------------------------ approximation
def g1_cubic(Q):
    """(cubic points, delta0, delta1) of the L2-optimal G1 reduction (p >= 4)."""
    Q = np.asarray(Q, dtype=np.float64)
    p = len(Q) - 1

    def mk(d0, d1):
        c = p / 3.0
        return np.array([Q[0], Q[0] + c * (Q[1] - Q[0]) * d0,
                         Q[p] - c * (Q[p] - Q[p - 1]) * d1, Q[p]])

    t0 = Q[1] - Q[0]
    t1 = Q[p] - Q[p - 1]
    ext = Q.max(axis=0) - Q.min(axis=0)
    tiny = 1e-12 * max(float(np.linalg.norm(ext)), 1e-300)
    if np.linalg.norm(t0) <= tiny or np.linalg.norm(t1) <= tiny:
        return mk(1.0, 1.0), 1.0, 1.0
    Gm = gram(3, p)
    G3 = gram(3, 3)
    ends = np.array([Q[0], Q[0], Q[p], Q[p]])
    V1 = Gm[1] @ Q - G3[1] @ ends
    V2 = Gm[2] @ Q - G3[2] @ ends
    c = p / 3.0
    a11 = G3[1, 1] * c * float(t0 @ t0)
    a12 = -G3[1, 2] * c * float(t1 @ t0)
    a21 = G3[2, 1] * c * float(t0 @ t1)
    a22 = -G3[2, 2] * c * float(t1 @ t1)
    r1 = float(V1 @ t0)
    r2 = float(V2 @ t1)
    det = a11 * a22 - a12 * a21
    if abs(det) <= 1e-12 * (abs(a11 * a22) + abs(a12 * a21)):
        return mk(1.0, 1.0), 1.0, 1.0
    d0 = (r1 * a22 - a12 * r2) / det
    d1 = (a11 * r2 - a21 * r1) / det
    return mk(d0, d1), float(d0), float(d1)


def l2_error(Q, R):
    p = len(Q) - 1
    e = (np.einsum("id,ij,jd->", Q, gram(p, p), Q)
         - 2.0 * np.einsum("id,ij,jd->", Q, gram(p, 3), R)
         + np.einsum("id,ij,jd->", R, gram(3, 3), R))
    return max(float(e), 0.0)


def elevate(P, target):
    P = np.asarray(P, dtype=np.float64)
    while len(P) - 1 < target:
        p = len(P) - 1
        out = np.empty((p + 2, P.shape[1]))
        out[0] = P[0]
        for i in range(1, p + 1):
            w = i / (p + 1.0)
            out[i] = w * P[i - 1] + (1.0 - w) * P[i]
        out[p + 1] = P[p]
        P = out
    return P


def max_error(P, piv, Q, oiv, samples):
    us = np.linspace(0.0, 1.0, samples)
    ts = piv[0] + us * (piv[1] - piv[0])
    vs = (ts - oiv[0]) / (oiv[1] - oiv[0])
    err = np.linalg.norm(design(3, us) @ P - design(len(Q) - 1, vs) @ Q, axis=1)
    mx = float(err.max())
    return mx, us[err >= mx - 1e-12]


def restrict(Q, a, b):
    n = len(Q) - 1
    if a > 0.0:
        Q = split_matrices(a, n)[1] @ Q
        b = (b - a) / (1.0 - a)
    if b < 1.0:
        Q = split_matrices(b, n)[0] @ Q
    return Q


class DepthError(Exception):
    pass


def approximate(segments, tol, loop_samples=64, verify_samples=1024, max_depth=32):
    """[(points, (ta, tb))] -> sorted [(cubic points, (ta, tb), measured error)]."""
    done = []
    work = []
    origin = []
    for Q, iv in segments:
        Q = np.asarray(Q, dtype=np.float64)
        p = len(Q) - 1
        if p <= 2:
            done.append((elevate(Q, 3), iv, 0.0))
        elif p == 3:
            done.append((Q, iv, 0.0))
        else:
            origin.append((Q, iv))
            work.append((len(origin) - 1, 0.0, 1.0, g1_cubic(Q)[0], 0))
    while work:
        nxt = []
        for k, la, lb, P, depth in work:
            Q, (oa, ob) = origin[k]
            piv = (oa + la * (ob - oa), oa + lb * (ob - oa))
            mx, at = max_error(P, piv, Q, (oa, ob), loop_samples)
            if mx <= tol:
                mx2, at2 = max_error(P, piv, Q, (oa, ob), verify_samples)
                if mx2 <= tol:
                    done.append((P, piv, mx2))
                    continue
                at, mx = at2, mx2
            if depth >= max_depth:
                raise DepthError(f"tolerance {tol} not reached on {piv}")
            zs = [z for z in at if 1e-9 < z < 1.0 - 1e-9] or [0.5]
            cuts = [la] + [la + z * (lb - la) for z in zs] + [lb]
            pins = [de_casteljau(Q, c) for c in cuts[1:-1]]
            for j in range(len(cuts) - 1):
                child = np.array(g1_cubic(restrict(Q, cuts[j], cuts[j + 1]))[0])
                if j > 0:
                    child[0] = pins[j - 1]
                if j < len(cuts) - 2:
                    child[3] = pins[j]
                nxt.append((k, cuts[j], cuts[j + 1], child, depth + 1))
        work = nxt
    done.sort(key=lambda c: c[1][0])
    return done


def prepare(p, knots, ctrl, tol=1e-4):
    """The packed arrays of project.prepare_curve (project.py:225-238)."""
    cubics = approximate(decompose(p, knots, ctrl), tol)
    S = len(cubics)
    d = np.asarray(ctrl).shape[1]
    seg_pts = np.empty((S, 4, d))
    seg_ta = np.empty(S)
    seg_tb = np.empty(S)
    for i, (P, (a, b), _) in enumerate(cubics):
        seg_pts[i] = P
        seg_ta[i], seg_tb[i] = a, b
    seam_t = np.concatenate(([seg_ta[0]], seg_tb))
    seam_pt = np.concatenate((seg_pts[:1, 0, :], seg_pts[:, 3, :]))
    return dict(seg_pts=seg_pts, seg_ta=seg_ta, seg_tb=seg_tb, seam_t=seam_t, seam_pt=seam_pt,
                cubics=cubics)


# ---------------------------------------------------------- curve evaluation
def eval_curve(p, knots, ctrl, ts):
    """Curve points by the raw Cox-de Boor recursion (oracle.py:13-52)."""
    knots = np.asarray(knots, dtype=np.float64)
    ctrl = np.asarray(ctrl, dtype=np.float64)
    ts = np.asarray(ts, dtype=np.float64)
    nb = len(knots) - 1
    N = np.zeros((len(ts), nb))
    last = None
    for i in range(nb):
        if knots[i] < knots[i + 1]:
            N[:, i] = (knots[i] <= ts) & (ts < knots[i + 1])
            last = i
    end = ts == knots[-1]
    if np.any(end) and last is not None:
        N[end] = 0.0
        N[end, last] = 1.0
    for j in range(1, p + 1):
        M = np.zeros((len(ts), nb - j))
        for i in range(nb - j):
            d1 = knots[i + j] - knots[i]
            if d1 > 0.0:
                M[:, i] += (ts - knots[i]) / d1 * N[:, i]
            d2 = knots[i + j + 1] - knots[i + 1]
            if d2 > 0.0:
                M[:, i] += (knots[i + j + 1] - ts) / d2 * N[:, i + 1]
        N = M
    return N[:, : ctrl.shape[0]] @ ctrl


# ------------------------------------------------------ synthetic workloads
def clamped_uniform_curve(rng, p, n, dim):
    """_fixtures.random_clamped_curve(rng, p, n, dim, uniform_knots=True)
    (_fixtures.py:22-59): uniform interior knots, momentum random-walk net
    normalised to the unit box.  Returns (p, knots, ctrl)."""
    interior = n - p - 1
    mid = np.linspace(0.0, 1.0, interior + 2)[1:-1]
    knots = np.concatenate((np.zeros(p + 1), mid, np.ones(p + 1)))
    if n > 2:
        pts = np.zeros((n, dim))
        v = rng.normal(size=dim)
        v /= np.linalg.norm(v)
        for i in range(1, n):
            v = v + 0.55 * rng.normal(size=dim)
            v /= np.linalg.norm(v)
            pts[i] = pts[i - 1] + v
        lo = pts.min(axis=0)
        span = np.maximum(pts.max(axis=0) - lo, 1e-9)
        ctrl = (pts - lo) / span
    else:
        ctrl = rng.uniform(0.0, 1.0, (n, dim))
    return p, knots, ctrl
