"""CPU ORACLE for surfaces -- test infrastructure only (see __init__.py).

* decompose(pu, pv, ku, kv, net): Bezier patches by the reference's
  per-span curve decomposition (decompose.py:19-46, restated in prep.py)
  applied along v for every row, then along u for every column -- the
  tensor-product use SURVEY.md 8(c) prescribes.
* eval_surface: tensor Cox-de Boor (prep.eval_curve per direction).
* dense_truth: a dense-grid global search per patch (the oracle.py:95-128
  recipe -- grid, then local refinement -- in two parameters), used to check
  that the seeded-Newton minimiser of mrep_surface_oracle.c is global.
"""

import numpy as np

from . import prep as P


def decompose(pu, pv, ku, kv, net):
    """-> patch_pts [nus][nvs][pu+1][pv+1][3], patch_iv [nus][nvs][4]."""
    net = np.asarray(net, dtype=np.float64)
    nu = net.shape[0]
    rows = [P.decompose(pv, kv, net[r]) for r in range(nu)]
    nvs = len(rows[0])
    R = np.array([[seg[0] for seg in row] for row in rows])  # [nu][nvs][pv+1][3]
    cols = {}
    for j in range(nvs):
        for c in range(pv + 1):
            cols[j, c] = P.decompose(pu, ku, R[:, j, c])
    nus = len(cols[0, 0])
    pts = np.empty((nus, nvs, pu + 1, pv + 1, 3))
    iv = np.empty((nus, nvs, 4))
    for j in range(nvs):
        for c in range(pv + 1):
            for i, (Q, (a, b)) in enumerate(cols[j, c]):
                pts[i, j, :, c] = Q
                iv[i, j, 0], iv[i, j, 1] = a, b
        iv[:, j, 2], iv[:, j, 3] = rows[0][j][1]
    return pts, iv


def eval_surface(pu, pv, ku, kv, net, uv):
    net = np.asarray(net, dtype=np.float64)
    out = np.empty((len(uv), 3))
    for i, (u, v) in enumerate(np.atleast_2d(uv)):
        col = np.array([P.eval_curve(pv, kv, net[r], np.array([v]))[0] for r in range(net.shape[0])])
        out[i] = P.eval_curve(pu, ku, col, np.array([u]))[0]
    return out


def _bern(p, u):
    from math import comb
    u = np.asarray(u, dtype=np.float64)
    return np.stack([comb(p, a) * u ** a * (1 - u) ** (p - a) for a in range(p + 1)], axis=-1)


def dense_truth(patch_pts, pu, pv, q, grid=65, refine=3):
    """Global minimum distance of q over all patches by a dense grid search
    (grid x grid samples per patch; on the 6 best patches, rounds of a 9x9
    grid around the best sample, the window shrinking 4x per round).
    Returns (dist, patch)."""
    pts = np.asarray(patch_pts, dtype=np.float64).reshape(-1, pu + 1, pv + 1, 3)
    g = np.linspace(0.0, 1.0, grid)
    Bu, Bv = _bern(pu, g), _bern(pv, g)
    S = np.einsum("ia,jc,pacx->pijx", Bu, Bv, pts)  # [np][grid][grid][3]
    d2 = ((S - q) ** 2).sum(-1)
    best = np.inf
    bp = -1
    for p in np.argsort(d2.reshape(len(pts), -1).min(1))[:6]:
        k = np.argmin(d2[p])
        u, v = g[k // grid], g[k % grid]
        h = 1.0 / (grid - 1)
        for _ in range(refine + 9):
            us = np.clip(u + h * np.linspace(-1, 1, 9), 0, 1)
            vs = np.clip(v + h * np.linspace(-1, 1, 9), 0, 1)
            Ss = np.einsum("ia,jc,acx->ijx", _bern(pu, us), _bern(pv, vs), pts[p])
            dd = ((Ss - q) ** 2).sum(-1)
            k = np.argmin(dd)
            u, v = us[k // 9], vs[k % 9]
            h /= 4.0
        dmin = float(np.sqrt(dd.min()))
        if dmin < best:
            best, bp = dmin, int(p)
    return best, bp
