"""pytest plugin: run the reference's own test suite against this package.

    python -m pytest -p splinemat_alias <dir holding the reference tests>

(scripts/run_ref_suite.sh stages the tests from /root/reference into the
git-ignored build/ref_suite/ and runs them on the GPU box.)  Every
``splinemat`` module a test imports is mapped onto the B200 package; the
reference's backend shim reports its numpy lane (``USING_NUMBA = False``),
which is what the jit-vs-python comparisons of tests/test_kernels.py skip on:
this package has exactly one backend, the sm_100a library.
"""
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_2504_11498_b200 as pkg  # noqa: E402
from paper_2504_11498_b200 import (  # noqa: E402
    _kernels, basis, cli, core, decompose, distance, fixtures, project, reduce_approx, selftest,
    verify)

_accel = types.ModuleType("splinemat._accel")
_accel.USING_NUMBA = False
_accel.njit = lambda *a, **k: (a[0] if a and callable(a[0]) else (lambda f: f))

ALIASES = {
    "splinemat": pkg, "splinemat._fixtures": fixtures, "splinemat.oracle": verify,
    "splinemat._kernels": _kernels, "splinemat._accel": _accel, "splinemat.basis": basis,
    "splinemat.cli": cli, "splinemat.core": core, "splinemat.decompose": decompose,
    "splinemat.distance": distance, "splinemat.project": project,
    "splinemat.reduce_approx": reduce_approx, "splinemat.selftest": selftest,
}
sys.modules.update(ALIASES)
for name, mod in ALIASES.items():
    if "." in name:
        setattr(pkg, name.split(".", 1)[1], mod)
