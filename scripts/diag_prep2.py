"""Time the pieces of prepare_curve_set (cfg3)."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_11498_b200 import _lib as L  # noqa: E402
from paper_2504_11498_b200.batch import prepare_curve_set  # noqa: E402
from paper_2504_11498_b200.decompose import DeviceCurves, decompose_device  # noqa: E402
from paper_2504_11498_b200.fixtures import mixed_curve_batch  # noqa: E402
from paper_2504_11498_b200.reduce_approx import approximate_device  # noqa: E402

curves = mixed_curve_batch(10000)
prepare_curve_set(curves[:50])
for rep in range(3):
    torch.cuda.synchronize()
    T = [time.perf_counter()]
    dec = decompose_device(DeviceCurves(curves))
    torch.cuda.synchronize()
    T.append(time.perf_counter())
    res = approximate_device(dec["rows"], dec["row_ofs"], dec["iv"], dec["curve"], dec["nseg"], 3,
                             1e-4, 4096 * len(curves))
    torch.cuda.synchronize()
    T.append(time.perf_counter())
    pts, iv, err, cid = res.fetch()
    counts = torch.bincount(cid.to(torch.int64), minlength=len(curves))
    ofs = np.concatenate(([0], np.cumsum(L.to_host(counts)))).astype(np.int64)
    ta = iv[:, 0].contiguous()
    tb = iv[:, 1].contiguous()
    torch.cuda.synchronize()
    T.append(time.perf_counter())
    h = ctypes.c_void_p()
    L.check(L.lib().mrep_curveset_create_dev(L.ptr(pts), L.ptr(ta), L.ptr(tb),
                                             ctypes.c_void_p(ofs.ctypes.data), len(curves), 3,
                                             L.stream_ptr(), ctypes.byref(h)))
    torch.cuda.synchronize()
    T.append(time.perf_counter())
    a, b, c = L.to_host(pts), L.to_host(ta), L.to_host(tb)
    T.append(time.perf_counter())
    L.lib().mrep_curveset_free(h)
    d = np.diff(T) * 1e3
    print("decompose %.0f approx %.0f fetch %.0f set_create %.0f to_host %.0f ms" % tuple(d))
