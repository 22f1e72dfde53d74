"""ctypes binding of libmrep.so (the C ABI declared in include/mrep.h).

This replaces the reference's backend shim ``_accel.py`` (``_accel.py:10-38``):
there is exactly one backend, the sm_100a library, and no CPU fallback.  If
the library is missing or no CUDA device is visible, every numeric entry point
raises ``RuntimeError`` instead of silently computing on the host.

Device memory and streams come from PyTorch (plumbing only): arguments are
torch tensors on ``cuda`` and their ``data_ptr()`` is handed to the C ABI
together with the current stream handle.
"""

import atexit
import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MREP_LIB: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("MREP_LIB") or os.path.join(_HERE, "libmrep.so")

MREP_SCREEN = 1
MREP_STATS = 2
MREP_NO_SORT = 4
MREP_FUSED = 8
MREP_TIMING = 16
MREP_PACKET = 32
MREP_PER_LANE = 64
MREP_GROUP = 128
MREP_CELLS = 256
MREP_CAND_EXACT = 512
MREP_CAND_CELLS = 1024
NUM_COUNTERS = 8
(CNT_PAIRS, CNT_SURVIVORS, CNT_CLIP_ITERS, CNT_SEAMS, CNT_BOXES, CNT_PASS2, CNT_HULL_MISS,
 CNT_UNCERTAIN) = range(8)

_lib = None
_lock = threading.Lock()

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_dbl = ctypes.c_double
_u32 = ctypes.c_uint

_SIGS = {
    "mrep_last_error": ([], ctypes.c_char_p),
    "mrep_version": ([], _i32),
    "mrep_last_stage_times": ([_vp, _i32], _i32),
    "mrep_fp64_peak": ([_vp], _i32),
    "mrep_dmma_peak": ([_vp], _i32),
    "mrep_host_release": ([], _i32),
    "mrep_device_count": ([], _i32),
    "mrep_table_bytes": ([_i64], _i64),
    "mrep_table_pack": ([_vp, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp], _i32),
    "mrep_project": ([_vp, _i64, _i32, _vp, _i64, _dbl, _i32, _i32, _u32, _vp, _vp, _vp, _vp,
                      _vp, _vp, _vp, _vp, _vp], _i32),
    "mrep_project_host": ([_vp, _i64, _i32, _vp, _i64, _dbl, _i32, _u32, _vp, _vp, _vp, _vp,
                           _vp, _vp], _i32),
    "mrep_project_block": ([_vp, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _i64, _dbl, _i32, _i32,
                            _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i32),
    "mrep_table_create": ([_vp, _vp, _vp, _vp, _vp, _i64, _i32, _vp], _i32),
    "mrep_table_free": ([_vp], _i32),
    "mrep_project_block_host": ([_vp, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _i64, _dbl, _i32, _i32,
                                 _vp, _vp, _vp, _vp, _vp, _vp], _i32),
    "mrep_curveset_create_dev": ([_vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp], _i32),
    "mrep_curveset_create": ([_vp, _vp, _vp, _vp, _i64, _i32, _vp], _i32),
    "mrep_curveset_free": ([_vp], _i32),
    "mrep_curveset_cells_build": ([_vp, _i32, _i64, _vp, _vp], _i32),
    "mrep_curveset_info": ([_vp, _vp, _vp, _vp, _vp], _i32),
    "mrep_project_batch": ([_vp, _vp, _vp, _i64, _dbl, _i32, _u32, _vp, _vp, _vp, _vp, _vp, _vp,
                            _vp], _i32),
    "mrep_project_batch_host": ([_vp, _vp, _vp, _i64, _dbl, _i32, _u32, _vp, _vp, _vp, _vp, _vp,
                                 _vp], _i32),
    "mrep_surface_table_bytes": ([_i64, _i32, _i32], _i64),
    "mrep_surface_table_pack": ([_vp, _vp, _i64, _i64, _i32, _i32, _vp, _vp], _i32),
    "mrep_project_surface": ([_vp, _i64, _i32, _i32, _vp, _i64, _u32, _vp, _vp, _vp, _vp, _vp,
                              _vp, _vp], _i32),
    "mrep_project_surface_host": ([_vp, _i64, _i32, _i32, _vp, _i64, _u32, _vp, _vp, _vp, _vp,
                                   _vp, _vp], _i32),
    "mrep_eval_surface": ([_i32, _i32, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _vp, _i64, _vp, _vp],
                          _i32),
    "mrep_oracle_project_batch": ([_i32, _vp, _i64, _vp, _i64, _i32, _vp, _vp, _i64, _vp, _i64,
                                   _vp, _vp, _vp], _i32),
    "mrep_synth_walk": ([_vp, _vp, _i64, _i32, _vp], _i32),
    "mrep_cells_bytes": ([_vp, _i64, _i32, _i32, _vp], _i64),
    "mrep_cells_build": ([_vp, _i64, _i32, _i32, _vp, _i64, _vp], _i32),
    "mrep_cand_cells_bytes": ([_vp, _i64, _i32, _i32, _vp], _i64),
    "mrep_cand_cells_build": ([_vp, _i64, _i32, _i32, _vp, _i64, _vp], _i32),
    "mrep_cand_cells_create": ([_vp, _i64, _i32, _i32, _vp], _i32),
    "mrep_surface_cells_bytes": ([_vp, _i64, _i32, _i32, _i32, _vp], _i64),
    "mrep_surface_cells_build": ([_vp, _i64, _i32, _i32, _i32, _vp, _i64, _vp], _i32),
    "mrep_knot_span": ([_vp, _i64, _i32, _vp, _i64, _vp, _vp], _i32),
    "mrep_knot_span_batch": ([_vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp], _i32),
    "mrep_quartic_roots": ([_vp, _i64, _vp, _vp, _vp], _i32),
    "mrep_newton_quartic_roots": ([_vp, _i64, _vp, _vp, _vp], _i32),
    "mrep_distance_poly": ([_vp, _vp, _i64, _i32, _vp, _vp], _i32),
    "mrep_restrict_ordinates": ([_vp, _vp, _vp, _i64, _vp, _vp], _i32),
    "mrep_eval_ordinates": ([_vp, _vp, _i64, _vp, _vp], _i32),
    "mrep_hull_cross": ([_vp, _i64, _vp, _vp, _vp], _i32),
    "mrep_clip_root": ([_vp, _i64, _dbl, _i32, _vp, _vp, _vp, _vp, _vp], _i32),
    "mrep_ordinates_op": ([_i32, _vp, _i32, _i64, _vp, _vp, _dbl, _i32, _vp, _vp, _vp, _vp, _vp],
                          _i32),
    "mrep_cubic_points": ([_vp, _vp, _i64, _i32, _vp, _vp], _i32),
    "mrep_rebase": ([_vp, _i64, _vp, _vp], _i32),
    "mrep_decompose_plan": ([_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp], _i32),
    "mrep_decompose": ([_vp, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _i64, _vp, _vp, _vp,
                        _vp, _vp, _vp], _i32),
    "mrep_eval_bezier": ([_vp, _i32, _i32, _vp, _i64, _vp, _vp], _i32),
    "mrep_basis_rows": ([_i32, _vp, _i64, _vp, _i64, _vp, _vp], _i32),
    "mrep_eval_curve": ([_i32, _vp, _i64, _vp, _i64, _i32, _vp, _i64, _vp, _vp], _i32),
    "mrep_approx_run": ([_vp, _vp, _vp, _vp, _i64, _i32, _dbl, _i64, _i32, _i32, _i32, _i32,
                         _vp, _vp], _i32),
    "mrep_approx_count": ([_vp], _i64),
    "mrep_approx_fetch": ([_vp, _vp, _vp, _vp, _vp, _vp], _i32),
    "mrep_approx_num_levels": ([_vp], _i32),
    "mrep_approx_level_sizes": ([_vp, _i32, _vp, _vp], _i32),
    "mrep_approx_level_fetch": ([_vp, _i32, _vp, _vp, _vp, _vp, _vp], _i32),
    "mrep_approx_free": ([_vp], None),
    "mrep_span_basis": ([_vp, _i32, _i32, _dbl, _vp, _vp], _i32),
    "mrep_reduce_g1": ([_vp, _i32, _i32, _i64, _vp, _vp, _vp, _vp], _i32),
    "mrep_max_error": ([_vp, _dbl, _dbl, _vp, _i32, _i32, _dbl, _dbl, _i32, _vp, _vp, _vp], _i32),
    "mrep_elevate": ([_vp, _i32, _i32, _i32, _vp, _vp], _i32),
    "mrep_split_cubic": ([_vp, _i32, _dbl, _i32, _dbl, _dbl, _vp, _i32, _dbl, _dbl, _vp, _vp,
                          _vp], _i32),
}


def exported_symbols():
    """Every C entry point include/mrep.h declares (checked by the CPU tests)."""
    return list(_SIGS)


def load_library(path=LIB_PATH):
    """dlopen libmrep.so and bind the signatures (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"libmrep.so not found at {path}; build it with "
                "`python -m paper_2504_11498_b200._build` (there is no CPU fallback)")
        L = ctypes.CDLL(path)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        atexit.register(_release_at_exit)
        return L


def _torch():
    import torch
    return torch


def _release_at_exit():
    # free the host-call pipeline contexts (pinned + device staging buffers)
    # while the CUDA runtime is still up; nothing to do if CUDA never started
    try:
        import sys
        torch = sys.modules.get("torch")
        if _lib is not None and torch is not None and torch.cuda.is_initialized():
            _lib.mrep_host_release()
    except Exception:
        pass


def lib():
    """The loaded library, after checking a CUDA device is present."""
    L = load_library()
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2504_11498_b200 needs a CUDA device (sm_100a); "
                           "no CPU fallback exists")
    return L


def check(rc):
    if rc != 0:
        msg = _lib.mrep_last_error().decode() if _lib is not None else ""
        raise RuntimeError(f"libmrep error {rc}: {msg}")


def stream_ptr():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def device():
    return _torch().device("cuda", _torch().cuda.current_device())


def to_dev(a, dtype=None):
    """numpy / torch -> contiguous cuda tensor (float64 by default)."""
    torch = _torch()
    dtype = dtype or torch.float64
    if isinstance(a, torch.Tensor):
        return a.to(device=device(), dtype=dtype).contiguous()
    arr = np.ascontiguousarray(a)
    if not arr.flags.writeable:  # read-only inputs (as_readonly): torch wants a writable view
        arr = arr.copy()
    return torch.from_numpy(arr).to(device=device(), dtype=dtype, non_blocking=False).contiguous()


def empty(shape, dtype=None):
    torch = _torch()
    return torch.empty(shape, dtype=dtype or torch.float64, device=device())


def to_host(t):
    return t.detach().cpu().numpy()
