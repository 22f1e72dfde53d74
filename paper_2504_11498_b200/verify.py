"""Independent verification helpers -- the reference's oracle.py API surface
(oracle.py:45-160), evaluated on the GPU.

eval_de_boor_many / eval_de_boor: Cox-de Boor evaluation (mrep_eval_curve).
"""

import numpy as np

from . import _lib as L
from .core import BSplineCurve, DomainError


def eval_de_boor_many(curve: BSplineCurve, ts) -> np.ndarray:
    """Curve points at an array of parameters (oracle.py:45-52)."""
    ts = np.ascontiguousarray(np.asarray(ts, dtype=np.float64).reshape(-1))
    lo, hi = curve.domain
    if np.any(ts < lo) or np.any(ts > hi):
        raise DomainError(f"parameter outside domain [{lo}, {hi}]")
    d = curve.dimension
    kn = L.to_dev(curve.knots.knots)
    cp = L.to_dev(curve.control_points)
    td = L.to_dev(ts)
    out = L.empty((len(ts), d))
    if len(ts):
        L.check(L.lib().mrep_eval_curve(curve.degree, L.ptr(kn), len(curve.knots.knots),
                                        L.ptr(cp), curve.control_points.shape[0], d, L.ptr(td),
                                        len(ts), L.ptr(out), L.stream_ptr()))
    return L.to_host(out)


def eval_de_boor(curve: BSplineCurve, t: float) -> np.ndarray:
    return eval_de_boor_many(curve, [t])[0]
