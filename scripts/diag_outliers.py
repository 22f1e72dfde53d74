"""Per-step device times of the cfg2 projection (500 steps): outlier census,
with and without an nvidia-smi sampler running."""
import subprocess
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

wl = bench.SingleCurve("cfg2", 0, 1, 0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for i in range(5):
    flush.fill_(float(i + 1))
    wl.step()
torch.cuda.synchronize()


def run(tag, K=500):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(K)]
    for i in range(K):
        flush.fill_(float(i))
        ev[i][0].record()
        wl.step()
        ev[i][1].record()
    torch.cuda.synchronize()
    t = np.array([a.elapsed_time(b) for a, b in ev])
    big = np.nonzero(t > 1.2 * np.median(t))[0]
    print(tag, "median", round(float(np.median(t)), 4), "mean", round(float(t.mean()), 4),
          "outliers", len(big), [(int(i), round(float(t[i]), 2)) for i in big[:10]])


run("plain")
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader",
                      "-lms", "50"], stdout=subprocess.DEVNULL)
import time  # noqa: E402
time.sleep(0.5)
run("sampler")
p.terminate()
run("plain2")
