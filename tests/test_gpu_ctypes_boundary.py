"""The C ABI driven the way the reference would bind it: plain ctypes,
numpy host arrays, no GPU framework (INTEGRATION.md's stub)."""
import ctypes
import os

import numpy as np
import pytest

from conftest import ROOT, load_golden

pytestmark = pytest.mark.gpu

LIB = os.path.join(ROOT, "paper_2504_11498_b200", "libmrep.so")


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


@pytest.fixture(scope="module")
def lib(gpu):
    L = ctypes.CDLL(LIB)
    L.mrep_table_create.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_int64, ctypes.c_int,
                                                            ctypes.POINTER(ctypes.c_void_p)]
    L.mrep_table_free.argtypes = [ctypes.c_void_p]
    L.mrep_project_host.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                    ctypes.c_int64, ctypes.c_double, ctypes.c_int, ctypes.c_uint,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    L.mrep_project_block_host.argtypes = ([ctypes.c_void_p] * 5 + [ctypes.c_int64, ctypes.c_int,
                                          ctypes.c_void_p, ctypes.c_int64, ctypes.c_double,
                                          ctypes.c_int, ctypes.c_int] + [ctypes.c_void_p] * 6)
    return L


@pytest.mark.parametrize("name", ["cfg1_random", "cfg2", "deg5_2d", "kink"])
def test_project_block_host_is_the_reference_kernel(lib, name):
    z = load_golden(f"project_{name}.npz")
    S, _, d = z["seg_pts"].shape
    n = len(z["queries"])
    out = (np.empty(n), np.empty((n, d)), np.empty(n), np.empty(n, np.int64),
           np.zeros((n, 6), np.int64), np.empty(n))
    arrs = [np.ascontiguousarray(z[k]) for k in ("seg_pts", "seg_ta", "seg_tb", "seam_t", "seam_pt")]
    rc = lib.mrep_project_block_host(*[_p(a) for a in arrs], S, d,
                                     _p(np.ascontiguousarray(z["queries"])), n,
                                     float(z["clip_tol"]), int(z["max_iter"]), int(z["soundness"]),
                                     *[_p(o) for o in out])
    assert rc == 0
    assert np.all(np.abs(out[0] - z["t"]) <= 1e-6)
    assert np.all(np.abs(out[2] - z["dist"]) <= np.maximum(1e-9 * z["dist"], 1e-12))
    assert np.array_equal(out[3], z["cand"])
    assert np.array_equal(out[4], z["stats"])


def test_table_handle_and_host_projection(lib):
    z = load_golden("project_cfg2.npz")
    S, _, d = z["seg_pts"].shape
    arrs = [np.ascontiguousarray(z[k]) for k in ("seg_pts", "seg_ta", "seg_tb", "seam_t", "seam_pt")]
    h = ctypes.c_void_p()
    assert lib.mrep_table_create(*[_p(a) for a in arrs], S, d, ctypes.byref(h)) == 0
    q = np.ascontiguousarray(z["queries"])
    n = len(q)
    t, foot, dist = np.empty(n), np.empty((n, d)), np.empty(n)
    cand, seg = np.empty(n, np.int64), np.empty(n, np.int32)
    cnt = np.zeros(8, np.uint64)
    assert lib.mrep_project_host(h, S, d, _p(q), n, 1e-6, 8, 1, _p(t), _p(foot), _p(dist),
                                 _p(cand), _p(seg), _p(cnt)) == 0
    assert lib.mrep_table_free(h) == 0
    assert np.all(np.abs(t - z["t"]) <= 1e-6)
    assert np.all(np.abs(dist - z["dist"]) <= 1e-9 * z["dist"])
    assert cnt[0] > 0 and cnt[6] == 0  # pairs solved, no hull misses


@pytest.mark.parametrize("name", ["cfg1_random", "cfg2", "deg5_2d"])
def test_host_call_reference_cand_with_cand_index(lib, name):
    """flags MREP_SCREEN | MREP_CAND_EXACT return the
    reference's own cand; with mrep_cand_cells_create + MREP_CAND_CELLS too."""
    z = load_golden(f"project_{name}.npz")
    S, _, d = z["seg_pts"].shape
    n = len(z["queries"])
    arrs = [np.ascontiguousarray(z[k]) for k in ("seg_pts", "seg_ta", "seg_tb", "seam_t", "seam_pt")]
    h = ctypes.c_void_p()
    assert lib.mrep_table_create(*[_p(a) for a in arrs], S, d, ctypes.byref(h)) == 0
    lib.mrep_cand_cells_create.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                           ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
    q = np.ascontiguousarray(z["queries"])
    for flags, with_index in ((1 | 512, False), (1 | 512 | 1024, True)):
        cc = ctypes.c_void_p()
        if with_index:
            assert lib.mrep_cand_cells_create(h, S, d, 16, ctypes.byref(cc)) == 0
        out = (np.empty(n), np.empty((n, d)), np.empty(n), np.empty(n, np.int64),
               np.empty(n, np.int32))
        assert lib.mrep_project_host(h, S, d, _p(q), n, float(z["clip_tol"]), int(z["max_iter"]),
                                     flags, *[_p(o) for o in out], None) == 0
        assert np.array_equal(out[3], z["cand"]), (name, flags)
        assert np.all(np.abs(out[0] - z["t"]) <= 1e-6)
        if with_index:
            lib.mrep_table_free(cc)
    lib.mrep_table_free(h)
