"""End-to-end (host buffers) timing of the cfg2 projection for one pipeline
shape (MREP_E2E_CHUNK / MREP_E2E_SLOTS from the environment)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
wl = bench.SingleCurve(cfg, 0, 1, 0)
n = wl.n
q = torch.from_numpy(wl.q_host).pin_memory().numpy()
outs = [torch.empty(n, dtype=torch.float64).pin_memory().numpy(),
        torch.empty((n, 3), dtype=torch.float64).pin_memory().numpy(),
        torch.empty(n, dtype=torch.float64).pin_memory().numpy(),
        torch.empty(n, dtype=torch.int64).pin_memory().numpy(),
        torch.empty(n, dtype=torch.int32).pin_memory().numpy()]
import ctypes  # noqa: E402
from paper_2504_11498_b200 import _lib as L  # noqa: E402
lib = L.lib()
p = lambda a: ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)  # noqa
flags = 1 | wl.tab._cell_flag(n, True)  # what DeviceTable.project_host passes
for with_seg in (True, False):
    seg = outs[4] if with_seg else None
    for _ in range(3):
        lib.mrep_project_host(L.ptr(wl.tab.buf), wl.tab.S, 3, p(q), n, 1e-6, 8, flags, p(outs[0]),
                              p(outs[1]), p(outs[2]), p(outs[3]), p(seg), None)
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        lib.mrep_project_host(L.ptr(wl.tab.buf), wl.tab.S, 3, p(q), n, 1e-6, 8, flags, p(outs[0]),
                              p(outs[1]), p(outs[2]), p(outs[3]), p(seg), None)
        ts.append(time.perf_counter() - t0)
    print(f"{cfg} chunk={os.environ.get('MREP_E2E_CHUNK', 'def')} "
          f"slots={os.environ.get('MREP_E2E_SLOTS', 'def')} seg={with_seg}: "
          f"median {np.median(ts) * 1e3:.3f} ms  min {np.min(ts) * 1e3:.3f} ms")
