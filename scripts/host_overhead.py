"""Host-side cost of one small projection call (cfg1, 10^4 queries): wall
time of the ctypes call alone (no sync) vs the device time between events,
for the device entry (mrep_project) and the host-buffer entry."""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2504_11498_b200 import _lib as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
wl = bench.SingleCurve(cfg, 0, 1, 0)
n = wl.n
q = wl.q
flags = L.MREP_SCREEN | wl.tab._cell_flag(n, True)
outs = [torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty((n, 3), dtype=torch.float64, device="cuda"),
        torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.int64, device="cuda"),
        torch.empty(n, dtype=torch.int32, device="cuda")]
P = L.ptr
lib = L.lib()
args = (P(wl.tab.buf), wl.tab.S, 3, P(q), n, 1e-6, 8, 0, flags, P(outs[0]), P(outs[1]), P(outs[2]),
        P(outs[3]), P(outs[4]), None, None, None, L.stream_ptr())
for _ in range(20):
    lib.mrep_project(*args)
torch.cuda.synchronize()
host, dev = [], []
for _ in range(50):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    lib.mrep_project(*args)
    host.append((time.perf_counter() - t0) * 1e3)
    b.record()
    torch.cuda.synchronize()
    dev.append(a.elapsed_time(b))
print(f"{cfg} n={n} mrep_project: host enqueue {statistics.median(host):.4f} ms, device (events) {statistics.median(dev):.4f} ms")
# back-to-back calls: throughput once host and device overlap
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    lib.mrep_project(*args)
torch.cuda.synchronize()
print(f"  200 back-to-back calls: {(time.perf_counter() - t0) / 200 * 1e3:.4f} ms per call")
wl.pinned()
import numpy as np  # noqa: E402
onp = (np.empty(n), np.empty((n, 3)), np.empty(n), np.empty(n, dtype=np.int64), np.empty(n, dtype=np.int32))
pin = [torch.from_numpy(o).pin_memory() for o in onp]
onp = tuple(x.numpy() for x in pin)
for _ in range(10):
    wl.host(onp)
ts = []
for _ in range(50):
    t0 = time.perf_counter()
    wl.host(onp)
    ts.append((time.perf_counter() - t0) * 1e3)
print(f"  host-buffer call (mrep_project_host): {statistics.median(ts):.4f} ms")
