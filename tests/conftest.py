import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name))


def project_fixture_names():
    return sorted(os.path.basename(f)[len("project_"):-4]
                  for f in glob.glob(os.path.join(GOLDEN, "project_*.npz")))


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.lib()
    return oracle


@pytest.fixture(scope="session")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test ran without a CUDA device")
    from paper_2504_11498_b200 import _lib
    _lib.lib()
    return torch.device("cuda")


def oracle_spans(knots, p, t):
    """Knot span convention of core.py:108-112 on the host (numpy)."""
    knots = np.asarray(knots)
    return np.clip(np.searchsorted(knots, t, "right") - 1, p, len(knots) - p - 2)


def assert_parity(t, dist, seg, o, span=None, knots=None, degree=None, dist_floor=1e-12):
    """North-star bars against an oracle result dict o (oracle.project_block):
    t within 1e-6; distance within 1e-9 relative (absolute floor dist_floor);
    winning segment EXACT on every query whose segment the oracle finds
    unambiguous (o["tie"] == 0: no other segment's candidate within
    dmin + 2e-12); knot span exact unless a knot lies between the GPU's t and
    the oracle's (then both spans are the correct span of their own t).
    Returns the number of oracle-detected ties."""
    assert np.all(np.abs(t - o["t"]) <= 1e-6), float(np.abs(t - o["t"]).max())
    tol = np.maximum(1e-9 * o["dist"], dist_floor)
    assert np.all(np.abs(dist - o["dist"]) <= tol), float(np.abs(dist - o["dist"]).max())
    clear = o["tie"] == 0
    bad = np.nonzero(clear & (seg != o["seg"]))[0]
    assert bad.size == 0, f"{bad.size} segment mismatches outside ties, e.g. {bad[:5]}"
    if span is not None:
        ref = oracle_spans(knots, degree, o["t"])
        assert np.array_equal(oracle_spans(knots, degree, t), span)
        diff = np.nonzero(span != ref)[0]
        for i in diff:  # only where t and t_ref straddle a knot
            lo, hi = sorted((t[i], o["t"][i]))
            assert np.any((knots > lo) & (knots <= hi)), (i, t[i], o["t"][i])
    return int((~clear).sum())
