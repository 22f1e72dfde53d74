"""Benchmark: projected points/s for the M-rep projection path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mrep|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)

Workload (BASELINE.json configs[1], "cfg2"): 10^6 uniformly random points in
[0,1]^3 per GPU projected onto a degree-7 clamped B-spline with 512 control
points (seed 0, uniform knots; 510 cubics after the 1e-4 approximation).  One
step = one projection pass over the rank's 10^6 resident queries.  Inputs
(24 MB) and outputs fit in the 126 MB L2, so L2 is flushed (256 MB write)
before every timed step, outside the per-step CUDA-event window.

N > 1: queries are sharded (each rank its own 10^6, weak scaling), the
curve is prepared on every GPU (replicated table), and each step ends with
the north star's single exchange: a gather of (t, dist, segment id) to rank 0
over NCCL.

Reported next to the device value:
* e2e: the same metric through the reference-facing C-ABI call with host
  buffers (mrep_project_host: pinned query buffer in, host results out, H2D
  + kernel + D2H inside the timed step);
* roofline: the projection kernel's algorithmic FP64 flop rate (work counters
  x per-unit flop constants of SURVEY.md 8(d)) against a DFMA peak measured
  in the same run;
* cpu_baseline: the pinned C restatement of the reference kernel (oracle/) on
  all host cores over a bounded sample of the same workload.
--impl reference runs that CPU restatement as the reference arm (rank 0
only; the Python reference itself does not travel to the GPU box).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "projected points/sec (curve & surface, fp64) at 1/2/4/8 B200 vs CPU ref"
UNIT = "points/s"
N_PER_RANK = 1_000_000
# FP64 flop per unit of work (d = 3)
F_PAIR, F_CLIP, F_SEAM, F_BOX = 500.0, 650.0, 10.0, 10.0


def workload_config(n):
    return {"workload": "cfg2: 1e6 random points/GPU onto a degree-7 B-spline, 512 ctrl pts "
                        "(510 cubic Beziers after 1e-4 approximation)",
            "queries_per_gpu": n, "degree": 7, "control_points": 512, "tolerance": 1e-4,
            "clip_tol": 1e-6, "max_iterations": 8, "dim": 3,
            "l2": "flushed (256 MB write) before each timed step",
            "mode": "BVH-screened exact solve (t/dist/segment identical to brute force)"}


def make_curve():
    from oracle import prep as P
    return P.clamped_uniform_curve(np.random.default_rng(0), 7, 512, 3)


def make_queries(rank, n):
    return np.random.default_rng(1 + rank).uniform(0.0, 1.0, (n, 3))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def cpu_baseline(seg, queries, sample_n, workers):
    """The reference kernel restated in C (oracle/), all host cores."""
    import oracle
    q = queries[:sample_n]
    oracle.project_block(*seg, q[: min(2000, sample_n)], workers=workers)  # warm
    t0 = time.perf_counter()
    oracle.project_block(*seg, q, workers=workers)
    dt = time.perf_counter() - t0
    return sample_n / dt, dt


def prepared_arrays():
    """Segment table of the cfg2 curve, built by the GPU prep pipeline."""
    from paper_2504_11498_b200 import BSplineCurve, prepare_curve
    p, knots, ctrl = make_curve()
    curve = BSplineCurve(p, knots, ctrl)
    import torch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prep = prepare_curve(curve, 1e-4)
    torch.cuda.synchronize()
    return prep, (time.perf_counter() - t0) * 1e3


def run_reference(args, rank):
    if rank != 0:
        return
    import oracle
    from oracle import prep as P
    p, knots, ctrl = make_curve()
    pr = P.prepare(p, knots, ctrl, 1e-4)
    seg = (pr["seg_pts"], pr["seg_ta"], pr["seg_tb"], pr["seam_t"], pr["seam_pt"])
    cores = len(os.sched_getaffinity(0))
    sample = args.ref_sample
    q = make_queries(0, sample)
    for _ in range(args.warmup):
        oracle.project_block(*seg, q[: max(1000, sample // 10)], workers=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.project_block(*seg, q, workers=cores)
        times.append(time.perf_counter() - t0)
    ms = statistics.mean(times) * 1e3
    value = sample / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(N_PER_RANK), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{sample} of the cfg2 queries per step, brute force over "
                                       f"all 510 cubics (C restatement of _kernels._project_block, "
                                       f"bit-exact vs the reference), {cores} threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mrep", choices=["mrep", "reference"])
    ap.add_argument("--n", type=int, default=N_PER_RANK)
    ap.add_argument("--ref-sample", type=int, default=32768)
    ap.add_argument("--cpu-sample", type=int, default=65536)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dense", action="store_true", help="brute-force kernel (reference semantics)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2504_11498_b200 import _lib as L
    from paper_2504_11498_b200 import _device as D

    prep, prep_ms = prepared_arrays()
    tab = prep.table
    n = args.n
    q_host = make_queries(rank, n)
    q = torch.from_numpy(q_host).cuda()
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    counters = torch.zeros(L.NUM_COUNTERS, dtype=torch.int64, device="cuda")
    screen = not args.dense

    def step(cnt=None):
        return tab.project(q, screen=screen, counters=cnt)

    def gather(out):
        if world == 1:
            return
        t, dd, seg = out[0], out[2], out[4].to(torch.float64)
        pack = torch.stack([t, dd, seg], 1).contiguous()
        bufs = [torch.empty_like(pack) for _ in range(world)] if rank == 0 else None
        dist.gather(pack, bufs, dst=0)

    for _ in range(args.warmup):
        gather(step())
    torch.cuda.synchronize()

    # ---- timed device steps (inputs resident in HBM) ----
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kstarts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.fill_(float(i))
            starts[i].record(stream)
            kstarts[i].record(stream)
            out = step(counters if i == 0 else None)
            kends[i].record(stream)
            gather(out)
            ends[i].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    kern_ms = [s.elapsed_time(e) for s, e in zip(kstarts, kends)]
    ms = statistics.mean(step_ms)
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = world * n / (ms / 1e3)

    # ---- roofline of the projection kernel ----
    c = counters.cpu().numpy().astype(np.float64)
    flops = (F_PAIR * c[L.CNT_PAIRS] + F_CLIP * c[L.CNT_SURVIVORS] + F_SEAM * c[L.CNT_SEAMS]
             + F_BOX * c[L.CNT_BOXES])
    kms = statistics.mean(kern_ms)
    import ctypes
    peak = ctypes.c_double()
    L.check(L.lib().mrep_fp64_peak(ctypes.byref(peak)))
    achieved = flops / (kms / 1e3) / 1e12
    dense_equiv = (F_PAIR * 510 + F_SEAM * 511) * n / (kms / 1e3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("project_kernel_dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s",
                "frac": achieved / peak.value, "traffic": traffic,
                "peak_source": "DFMA microbenchmark measured in this run (mrep_fp64_peak); "
                               "MEASURED_PEAKS.json has no FP64 figure",
                "flop_model": "500/pair + 650/clipped survivor + 10/seam + 10/box test "
                              "(SURVEY.md 8(d), counters from the kernel)",
                "per_query": {"pairs": c[L.CNT_PAIRS] / n, "survivors": c[L.CNT_SURVIVORS] / n,
                              "seams": c[L.CNT_SEAMS] / n, "box_tests": c[L.CNT_BOXES] / n},
                "kernel_ms": kms,
                "dense_equivalent_tflops": dense_equiv,
                "hbm": {"bytes_per_query": 24 + 8 + 24 + 8 + 8 + 4,
                        "gbs": n * 76 / (kms / 1e3) / 1e9}}

    # ---- e2e: host buffers through the C ABI (H2D + kernel + D2H per step) ----
    q_pin = torch.from_numpy(q_host).pin_memory()
    outs = (torch.empty(n, dtype=torch.float64).pin_memory(),
            torch.empty((n, 3), dtype=torch.float64).pin_memory(),
            torch.empty(n, dtype=torch.float64).pin_memory(),
            torch.empty(n, dtype=torch.int64).pin_memory(),
            torch.empty(n, dtype=torch.int32).pin_memory())
    onp = tuple(o.numpy() for o in outs)
    qnp = q_pin.numpy()
    for _ in range(2):
        tab.project_host(qnp, out=onp, screen=screen)
    e2e_times = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tab.project_host(qnp, out=onp, screen=screen)
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = statistics.mean(e2e_times)
    if world > 1:
        tt = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e = {"value": world * n / e2e_s, "unit": UNIT, "h2d_bytes_per_step": n * 24,
           "d2h_bytes_per_step": n * (8 + 24 + 8 + 8 + 4),
           "path": "mrep_project_host (C ABI, pinned host buffers, 2-stream chunked pipeline)"}

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            seg = (prep.seg_pts, prep.seg_ta, prep.seg_tb, prep.seam_t, prep.seam_pt)
            cores = len(os.sched_getaffinity(0))
            v, dt = cpu_baseline(seg, q_host, args.cpu_sample, cores)
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                   "sample": f"first {args.cpu_sample} of the 1e6 queries, brute force over all "
                             f"510 cubics ({dt:.1f} s wall on {cores} threads); C restatement of "
                             f"_kernels._project_block, bit-exact vs the reference"}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": dict(workload_config(n),
                                                    parallelism=f"query-shard x{world}",
                                                    prep_ms=prep_ms),
                "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu,
                "gpu_launches": 2 * args.steps, "clocks": clocks.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
