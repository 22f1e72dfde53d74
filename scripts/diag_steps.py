"""Per-step device time vs host enqueue time of the bench step (diagnostic)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
wl = (bench.CurveSetWorkload if cfg == "cfg3" else bench.SingleCurve)(cfg, 0, 1, 0)
from paper_2504_11498_b200 import _lib as L  # noqa: E402
for name, fl in (("packet", L.MREP_PACKET), ("per-lane", L.MREP_PER_LANE), ("group", L.MREP_GROUP)):
    for _ in range(3):
        wl.step(extra_flags=fl)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        wl.step(extra_flags=fl)
    b.record()
    torch.cuda.synchronize()
    print(cfg, name, "ms/step %.3f" % (a.elapsed_time(b) / 20))
for _ in range(5):
    wl.step()
torch.cuda.synchronize()
st = torch.cuda.current_stream()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
host = []
for a, b in ev:
    t0 = time.perf_counter()
    a.record(st)
    wl.step()
    b.record(st)
    host.append((time.perf_counter() - t0) * 1e3)
torch.cuda.synchronize()
dev = [a.elapsed_time(b) for a, b in ev]
print(cfg, "device ms: median %.3f mean %.3f max %.3f" % (np.median(dev), np.mean(dev), np.max(dev)))
print(cfg, "host enqueue ms: median %.3f mean %.3f max %.3f" % (np.median(host), np.mean(host), np.max(host)))
# back-to-back with a sync each: pure GPU time with an idle host
dev2 = []
for a, b in ev[:20]:
    torch.cuda.synchronize()
    a.record(st)
    wl.step()
    b.record(st)
    torch.cuda.synchronize()
    dev2.append(a.elapsed_time(b))
print(cfg, "synced device ms: median %.3f" % np.median(dev2))
# graph capture of one step
g = torch.cuda.CUDAGraph()
s2 = torch.cuda.Stream()
s2.wait_stream(st)
with torch.cuda.stream(s2):
    wl.step()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s2):
        out = wl.step()
torch.cuda.synchronize()
gd = []
for a, b in ev[:30]:
    a.record(st)
    g.replay()
    b.record(st)
torch.cuda.synchronize()
gd = [a.elapsed_time(b) for a, b in ev[:30]]
print(cfg, "graph replay ms: median %.3f mean %.3f" % (np.median(gd), np.mean(gd)))
