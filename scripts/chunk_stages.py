"""Per-stage device times (MREP_TIMING, CUDA events inside the library) of
one cfg2 projection at several batch sizes, plus the whole call's event
time: where the fixed per-call latency goes."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2504_11498_b200 import _lib as L  # noqa: E402

wl = bench.SingleCurve("cfg2", 0, 1, 0)
names = ["sort", "traverse", "pairs", "clip", "select", "fallback", "cand"]
for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "65536,200000,1000000").split(",")]:
    q = wl.q[:n].contiguous()
    flags = wl.tab._cell_flag(n, True)
    outs = [torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty((n, 3), dtype=torch.float64, device="cuda"),
            torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.int64, device="cuda"),
            torch.empty(n, dtype=torch.int32, device="cuda")]
    P = L.ptr
    def call(extra=0):
        L.check(L.lib().mrep_project(P(wl.tab.buf), wl.tab.S, 3, P(q), n, 1e-6, 8, 0,
                                     L.MREP_SCREEN | flags | extra, P(outs[0]), P(outs[1]), P(outs[2]),
                                     P(outs[3]), P(outs[4]), None, None, None, L.stream_ptr()))
    for _ in range(5):
        call()
    ev = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); call(); b.record(); torch.cuda.synchronize()
        ev.append(a.elapsed_time(b))
    ev.sort()
    call(L.MREP_TIMING)
    torch.cuda.synchronize()
    buf = (ctypes.c_double * 8)()
    L.lib().mrep_last_stage_times(buf, 8)
    st = {names[i]: round(buf[i], 4) for i in range(7)}
    print(f"n={n}: call {ev[len(ev)//2]:.4f} ms (events, preallocated outputs, direct ctypes); stages {st} sum {sum(st.values()):.4f}", flush=True)
