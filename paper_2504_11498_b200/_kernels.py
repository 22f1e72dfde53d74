"""The reference's kernel-module entry points (``splinemat._kernels``,
/root/reference/pkg/src/splinemat/_kernels.py) bound to libmrep.

Same names and calling convention as the numba kernels -- caller-allocated
output arrays filled in place, no return value -- so code (and tests) that
reach into ``_kernels`` directly keep working: this is the reference-side
binding of the C ABI (include/mrep.h) that INTEGRATION.md describes.  Every
call runs on the GPU; there is no host implementation.

* ``_project_block`` (_kernels.py:369-502)   -> mrep_project_block (brute
  force with the reference's cand, stats and soundness)
* ``_quartic_block`` (_kernels.py:506-512)   -> mrep_quartic_roots
* ``_newton_quartic_block`` (_kernels.py:515-...) -> mrep_newton_quartic_roots
"""

import numpy as np

from . import _device as D


def _project_block(seg_pts, seg_ta, seg_tb, seam_t, seam_pt, queries, clip_tol, max_iter,
                   soundness_samples, out_t, out_foot, out_dist, out_cand, out_stats, out_sound):
    t, foot, dist, cand, stats, sound = D.project_block(
        seg_pts, seg_ta, seg_tb, seam_t, seam_pt, queries, float(clip_tol), int(max_iter),
        int(soundness_samples))
    out_t[...] = t
    out_foot[...] = foot
    out_dist[...] = dist
    out_cand[...] = cand
    out_stats[...] = stats
    out_sound[...] = sound


def _fill_roots(roots, counts, out_roots, out_counts):
    out_counts[...] = counts
    for k in range(4):  # rows keep their prior contents past each count, as the reference
        m = counts > k
        out_roots[m, k] = roots[m, k]


def _quartic_block(coeffs, out_roots, out_counts):
    roots, counts = D.quartic_roots(np.asarray(coeffs, dtype=np.float64))
    _fill_roots(roots, counts, out_roots, out_counts)


def _newton_quartic_block(coeffs, out_roots, out_counts):
    roots, counts = D.newton_quartic_roots(np.asarray(coeffs, dtype=np.float64))
    _fill_roots(roots, counts, out_roots, out_counts)
