"""Benchmark: projected points/s for the M-rep projection path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mrep|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)

`python bench.py --gpus N` (N > 1, no WORLD_SIZE in the environment) starts
its own N ranks under torch.distributed.run on 127.0.0.1; under torchrun the
world size must equal --gpus.

Workload (BASELINE.json configs[1], "cfg2"): 10^6 uniformly random points in
[0,1]^3 per GPU projected onto a degree-7 clamped B-spline with 512 control
points (seed 0, uniform knots; 510 cubics after the 1e-4 approximation).  One
step = one projection pass over the rank's 10^6 resident queries.  Inputs
(24 MB) and outputs fit in the 126 MB L2, so L2 is flushed (256 MB write)
before every timed step, outside the per-step CUDA-event window.

N > 1: queries are sharded (each rank its own 10^6, weak scaling), the
curve is prepared on every GPU (replicated table), and the north star's
single exchange -- a gather of (t, dist, segment id) to rank 0 over NCCL --
runs per query chunk (4 per step), each chunk's gather overlapping the next
chunk's projection.  --verify-gather checks the gathered result bitwise
against one projection of every rank's queries.

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
CHUNKS = 4  # N > 1: query chunks per step, each gathered while the next projects


def spawn_ranks(n):
    """Re-launch this command as n ranks under torch.distributed.run (one
    process per GPU, rendezvous on 127.0.0.1); returns the launcher's exit code."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)]
    # torchrun's parser would read `--n` as an ambiguous abbreviation of its own options
    for a in sys.argv[1:]:
        cmd.append("--queries-per-gpu" + a[3:] if a == "--n" or a.startswith("--n=") else a)
    return subprocess.call(cmd)


CONFIGS = {
    # BASELINE.json configs[0]: inversion of 1e4 on-curve points, degree 3, 64 ctrl
    "cfg1": dict(degree=3, ctrl=64, n=10_000, queries="on-curve", scaling="weak",
                 desc="cfg1: 1e4 on-curve points (inversion) onto a degree-3 B-spline, "
                      "64 ctrl pts (61 cubics)"),
    # configs[1]: the headline
    "cfg2": dict(degree=7, ctrl=512, n=1_000_000, queries="uniform", scaling="weak",
                 desc="cfg2: 1e6 random points/GPU onto a degree-7 B-spline, 512 ctrl pts "
                      "(510 cubic Beziers after 1e-4 approximation)"),
    # configs[2]: 1e4 curves, mixed degree 3-9, 8-2048 ctrl pts, 100 points per curve
    "cfg3": dict(degree="3-9", ctrl="8-2048", n=1_000_000, queries="uniform", scaling="weak",
                 curves=10_000, per_curve=100,
                 desc="cfg3: 1e6 random points/GPU, 100 per curve, onto a batch of 1e4 "
                      "B-splines (degree 3-9, 8-2048 ctrl pts, log-uniform), one batched call"),
    # configs[3]: 1e6 points onto a 64x64-net surface, bicubic and degree 5
    "cfg4": dict(degree=3, ctrl="64x64", n=1_000_000, queries="uniform", scaling="weak",
                 surface=True,
                 desc="cfg4: 1e6 random points/GPU onto a bicubic B-spline surface, 64x64 "
                      "control net (3721 Bezier patches)"),
    "cfg4q": dict(degree=5, ctrl="64x64", n=1_000_000, queries="uniform", scaling="weak",
                  surface=True,
                  desc="cfg4 (degree 5): 1e6 random points/GPU onto a biquintic B-spline "
                       "surface, 64x64 control net (3481 Bezier patches)"),
    # configs[4]: 1e8 points onto 1e5 cubics, query-sharded (strong scaling)
    "cfg5": dict(degree=3, ctrl=100_003, n=100_000_000, queries="uniform", scaling="strong",
                 desc="cfg5: 1e8 random points onto a degree-3 B-spline with 100003 ctrl pts "
                      "(1e5 cubics), sharded across GPUs"),
    # SURVEY.md 8(f) item 4 (not a BASELINE config): nearest-over-set
    "cfg6": dict(degree="3-9", ctrl="8-2048", curves=100, n=1_000_000, queries="uniform",
                 scaling="weak", nearest=True,
                 desc="cfg6 (8(f) nearest-over-set): 1e6 random points/GPU, each projected "
                      "onto the NEAREST of 100 mixed curves (degree 3-9, 8-2048 ctrl pts) "
                      "merged into one table"),
}


def workload_config(cfg, n):
    c = CONFIGS[cfg]
    return {"workload": c["desc"], "queries_per_gpu": n, "degree": c["degree"],
            "control_points": c["ctrl"], "tolerance": 1e-4, "clip_tol": 1e-6,
            "max_iterations": 8, "dim": 3, "queries": c["queries"],
            "l2": "flushed (256 MB write) before each timed step",
            "mode": ("BVH-screened per-patch seeded projected Newton (equal to the brute-force "
                     "surface oracle)" if c.get("surface") else
                     "BVH-screened exact solve (t/dist/segment identical to brute force)")}


def make_curve(cfg="cfg2"):
    """(degree, knots, ctrl): random_clamped_curve(default_rng(0), p, n, 3,
    uniform_knots=True) -- the reference fixture generator's call sequence."""
    from paper_2504_11498_b200.fixtures import random_clamped_curve
    c = CONFIGS[cfg]
    cv = random_clamped_curve(np.random.default_rng(0), c["degree"], c["ctrl"], 3,
                              uniform_knots=True)
    return cv.degree, np.array(cv.knots.knots), np.array(cv.control_points)


def make_queries(cfg, rank, n, curve=None):
    rng = np.random.default_rng(1 + rank)
    if CONFIGS[cfg]["queries"] == "on-curve":
        from paper_2504_11498_b200 import BSplineCurve, eval_de_boor_many
        p, knots, ctrl = curve
        return eval_de_boor_many(BSplineCurve(p, knots, ctrl),
                                 rng.uniform(knots[0], knots[-1], n))
    return rng.uniform(0.0, 1.0, (n, 3))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled (every 50 ms) while the
    timed region runs; the sampler is this process's own child, stopped by PID."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None
        self._t = None

    def _reader(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._reader, daemon=True)
            self._t.start()
            time.sleep(0.3)  # first sample before the timed work starts
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self._t.join(timeout=5)

    def summary(self):
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def cpu_time(jobs, workers):
    """The reference kernel restated in C (oracle/), all host cores, over a
    list of (seg arrays, queries) jobs; returns (queries, seconds).  Surface
    jobs run the surface oracle (brute force over every patch)."""
    import oracle

    def run(job, q):
        if isinstance(job, str) and job == "surface":
            prep, qq = q
            pu, pv = prep.surface.degree_u, prep.surface.degree_v
            oracle.surface_project(prep.patch_pts.reshape(-1, pu + 1, pv + 1, 3),
                                   prep.patch_iv.reshape(-1, 4), pu, pv, qq, workers=workers)
            return len(qq)
        oracle.project_block(*job, q, workers=workers)
        return len(q)

    job, q = jobs[0]
    if isinstance(job, str):
        run(job, (q[0], q[1][:16]))
    else:
        run(job, q[: min(200, len(q))])  # warm
    t0 = time.perf_counter()
    nq = 0
    for job, q in jobs:
        nq += run(job, q)
    return nq, time.perf_counter() - t0


def cand_pairs_tested(tab, q, S):
    """(query, cubic) pairs the exact-cand pass tests: every cubic without a
    cand cell index; with one, each query's cell list (every cubic outside
    the grid) -- the grid words of the table header (mrep_cand.cuh H_CC*)."""
    n = int(q.shape[0])
    if getattr(tab, "cand_cells", None) is None:
        return float(n) * S
    h = tab.buf[24:36].cpu().numpy()
    G, glo, ginv, ghi = int(h[1]), h[2:5], h[5:8], h[8:11]
    d = tab.d
    ncell = G ** d
    off = tab.cand_cells[: ncell + 1].cpu().numpy().astype(np.int64)
    qq = q.cpu().numpy()[:, :d]
    inside = np.all((qq >= glo[:d]) & (qq < ghi[:d]), axis=1)
    ci = np.clip(((qq - glo[:d]) * ginv[:d]).astype(np.int64), 0, G - 1)
    cell = ci[:, 0]
    for k in range(1, d):
        cell = cell * G + ci[:, k]
    ln = np.where(inside, off[cell + 1] - off[cell], S)
    return float(ln.sum())


def _prep_one(args):
    """oracle/prep.py prepare() of one curve (the reference's numpy
    decomposition + error-controlled approximation, restated): cubic count."""
    from oracle import prep as P
    p, knots, ctrl = args
    return len(P.prepare(p, knots, ctrl, 1e-4)["cubics"])


def prep_measure(wl, cfg, cpu_sample_s=8.0):
    """Subsystem 1 (decomposition + approximation + packing) on the GPU vs the
    oracle's numpy restatement of the reference preprocessing on host cores."""
    import torch
    from concurrent.futures import ProcessPoolExecutor
    from paper_2504_11498_b200 import BSplineCurve, prepare_curve, prepare_curve_set
    if cfg == "cfg3":
        curves = [(c.degree, np.asarray(c.knots.knots), np.asarray(c.control_points))
                  for c in wl.curves]
        reps, S = 2, wl.num_segments
        run = lambda: prepare_curve_set(wl.curves, 1e-4).free()  # noqa: E731
    else:
        curves = [wl.curve]
        reps, S = 5, wl.num_segments
        run = lambda: prepare_curve(BSplineCurve(*wl.curve), 1e-4)  # noqa: E731
    run()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    gpu_s = statistics.median(ts)
    # CPU: a stratified sample of the same curves, one process per core
    cores = len(os.sched_getaffinity(0))
    if len(curves) == 1:
        sample, desc = curves, "the same curve, single-threaded (one curve has one serial level loop)"
        cores_used = 1
    else:
        k = max(cores * 3, 16)
        idx = np.linspace(0, len(curves) - 1, k).astype(int)
        sample = [curves[i] for i in idx]
        desc = f"{k} of the {len(curves)} curves (evenly spaced), one process per core"
        cores_used = cores
    t0 = time.perf_counter()
    if cores_used == 1:
        nc = sum(_prep_one(c) for c in sample)
    else:
        with ProcessPoolExecutor(cores_used) as ex:
            nc = sum(ex.map(_prep_one, sample))
    cpu_s = time.perf_counter() - t0
    return {"what": "prepare_curve / prepare_curve_set: knot-insertion decomposition, G1 "
                    "reduction + error-controlled subdivision, packing (north-star subsystem 1)",
            "gpu_ms": gpu_s * 1e3, "cubics": int(S), "cubics_per_s": S / gpu_s,
            "cpu": {"cubics_per_s": nc / cpu_s, "cores": cores_used, "kind": "port",
                    "sample": f"{desc}: {nc} cubics in {cpu_s:.1f} s; oracle/prep.py, the "
                              f"reference's numpy preprocessing restated (bit-exact goldens)"},
            "kernels": "approx_eval_kernel / approx_child_kernel / decompose_kernel "
                       "(profiles/r02_prep_launch_shares.txt)"}


def _seg(prep):
    return (prep.seg_pts, prep.seg_ta, prep.seg_tb, prep.seam_t, prep.seam_pt)


class SingleCurve:
    """cfg1 / cfg2 / cfg5: one prepared curve, the rank's query shard."""

    def __init__(self, cfg, rank, world, n_override):
        import torch
        from paper_2504_11498_b200 import BSplineCurve, prepare_curve
        c = CONFIGS[cfg]
        self.cfg, self.n_override = cfg, n_override
        self.curve = make_curve(cfg)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        self.prep = prepare_curve(BSplineCurve(*self.curve), 1e-4)
        self.tab = self.prep.table
        torch.cuda.synchronize()
        self.prep_ms = (time.perf_counter() - t0) * 1e3
        # the dense-batch cell index is part of the prepared table (built
        # lazily by the first large batch; built here so prep_ms includes it)
        t0 = time.perf_counter()
        self.tab._cell_flag(max(c["n"], 1 << 20), True)
        torch.cuda.synchronize()
        self.cells_ms = (time.perf_counter() - t0) * 1e3
        if n_override:
            self.n = n_override
        elif c["scaling"] == "strong":
            from paper_2504_11498_b200.sharding import shard_range
            lo, hi = shard_range(c["n"], rank, world)
            self.n = hi - lo
        else:
            self.n = c["n"]
        self.n_total = c["n"] if c["scaling"] == "strong" and not n_override else world * self.n
        self.q_host = make_queries(cfg, rank, self.n, self.curve)
        self.q = torch.from_numpy(self.q_host).cuda()
        self.num_segments = self.prep.num_segments
        self.h2d = self.n * 24

    def step(self, counters=None, extra_flags=0, dense=False, sl=slice(None)):
        return self.tab.project(self.q[sl], screen=not dense, counters=counters,
                                extra_flags=extra_flags)

    def inputs(self, r, world):
        n = self.n
        if CONFIGS[self.cfg]["scaling"] == "strong" and not self.n_override:
            from paper_2504_11498_b200.sharding import shard_range
            lo, hi = shard_range(CONFIGS[self.cfg]["n"], r, world)
            n = hi - lo
        return (make_queries(self.cfg, r, n, self.curve),)

    def project_all(self, inputs, dense=False):
        import torch
        q = torch.from_numpy(np.concatenate([i[0] for i in inputs])).cuda()
        out = self.tab.project(q, screen=not dense)
        return out[0], out[2], out[4]

    def pinned(self):
        import torch
        self.q_pin = torch.from_numpy(self.q_host).pin_memory().numpy()

    def host(self, out, dense=False, extra_flags=0):
        # the reference-facing call returns (t, foot, dist, cand): no segment ids
        self.tab.project_host(self.q_pin, out=out[:4] + (None,), screen=not dense,
                              extra_flags=extra_flags)

    def cpu_jobs(self, sample):
        sample = max(256, min(sample, int(sample * 510 / self.num_segments)))
        if sample <= len(self.q_host):
            qs = self.q_host[:sample]
            desc = f"first {sample} of the {self.n} queries"
        else:  # small batch (cfg1): the whole batch, repeated to a timeable sample
            reps = -(-sample // len(self.q_host))
            qs = np.concatenate([self.q_host] * reps)
            desc = f"the {len(self.q_host)} queries x {reps}"
        desc += f", brute force over all {self.num_segments} cubics"
        return [(_seg(self.prep), qs)], desc


class CurveSetWorkload:
    """cfg3: 1e4 mixed curves prepared as one device set, 100 queries per
    curve in random order, one batched projection call per step."""

    def __init__(self, cfg, rank, world, n_override):
        import torch
        from paper_2504_11498_b200 import prepare_curve_set
        from paper_2504_11498_b200.fixtures import mixed_curve_batch
        c = CONFIGS[cfg]
        self.curves = mixed_curve_batch(c["curves"])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        self.cset = prepare_curve_set(self.curves, 1e-4)
        torch.cuda.synchronize()
        self.prep_ms = (time.perf_counter() - t0) * 1e3
        # per-curve cell indices (part of preparation, timed separately)
        t0 = time.perf_counter()
        gmax = int(os.environ.get("MREP_SET_GRID", "20"))
        budget = int(float(os.environ.get("MREP_SET_BUDGET_GB", "16")) * (1 << 30))
        self.cells_bytes = self.cset.build_cells(gmax, budget) if gmax > 0 else 0
        torch.cuda.synchronize()
        self.cells_ms = (time.perf_counter() - t0) * 1e3
        self.n = n_override or c["n"]
        self.n_total = world * self.n
        self.q_host, self.cid_host = self.inputs(rank, world)
        self.q = torch.from_numpy(self.q_host).cuda()
        self.cid = torch.from_numpy(self.cid_host).cuda()
        self.num_segments = self.cset.num_segments
        self.h2d = self.n * (24 + 4)

    def step(self, counters=None, extra_flags=0, dense=False, sl=slice(None)):
        return self.cset.project_device(self.q[sl], self.cid[sl], counters=counters,
                                        extra_flags=extra_flags)

    def inputs(self, r, world):
        rng = np.random.default_rng(1 + r)
        cid = (np.arange(self.n) % CONFIGS["cfg3"]["curves"]).astype(np.int32)
        rng.shuffle(cid)
        return rng.uniform(0.0, 1.0, (self.n, 3)), cid

    def project_all(self, inputs, dense=False):
        import torch
        q = torch.from_numpy(np.concatenate([i[0] for i in inputs])).cuda()
        cid = torch.from_numpy(np.concatenate([i[1] for i in inputs])).cuda()
        out = self.cset.project_device(q, cid)
        return out[0], out[2], out[4]

    def pinned(self):
        import torch
        self.q_pin = torch.from_numpy(self.q_host).pin_memory().numpy()
        self.cid_pin = torch.from_numpy(self.cid_host).pin_memory().numpy()

    def host(self, out, dense=False):
        self.cset.project_host(self.q_pin, self.cid_pin, out=out[:4] + (None,))

    def cpu_jobs(self, sample):
        stride = max(1, len(self.curves) // 50)
        jobs, nq, ns = [], 0, 0
        for c in range(0, len(self.curves), stride):
            pr = self.cset[c]
            m = self.cid_host == c
            jobs.append((_seg(pr), self.q_host[m]))
            nq += int(m.sum())
            ns += pr.num_segments
        desc = (f"{nq} queries of {len(jobs)} stratified curves (every {stride}th, {ns} cubics), "
                f"brute force per curve")
        return jobs, desc


class NearestWorkload:
    """cfg6: the first 100 curves of the cfg3 generator merged into one
    nearest-over-set table (nearest.py); every query against all of them."""

    def __init__(self, cfg, rank, world, n_override):
        import torch
        from paper_2504_11498_b200 import _lib as L, prepare_curve_set, prepare_nearest_set
        from paper_2504_11498_b200.fixtures import mixed_curve_batch
        c = CONFIGS[cfg]
        self.curves = mixed_curve_batch(c["curves"])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cset = prepare_curve_set(self.curves, 1e-4)
        self.preps = [cset[i] for i in range(len(self.curves))]
        self.nset = prepare_nearest_set(self.preps)
        self.tab = self.nset.table
        torch.cuda.synchronize()
        self.prep_ms = (time.perf_counter() - t0) * 1e3
        t0 = time.perf_counter()
        self.tab._cell_flag(max(c["n"], 1 << 20), True)
        torch.cuda.synchronize()
        self.cells_ms = (time.perf_counter() - t0) * 1e3
        self.n = n_override or c["n"]
        self.n_total = world * self.n
        self.q_host = np.random.default_rng(1 + rank).uniform(0.0, 1.0, (self.n, 3))
        self.q = torch.from_numpy(self.q_host).cuda()
        self.num_segments = int(self.nset.counts.sum())
        self.h2d = self.n * 24
        # per-query walks offer both seams of a cubic (nearest.py)
        self.mode = 0 if self.n >= 8 * self.tab.S else L.MREP_PER_LANE
        self.cpu_div = len(self.preps)  # the CPU sample runs every curve per query

    def step(self, counters=None, extra_flags=0, dense=False, sl=slice(None)):
        return self.tab.project(self.q[sl], counters=counters, extra_flags=extra_flags | self.mode)

    def inputs(self, r, world):
        return (np.random.default_rng(1 + r).uniform(0.0, 1.0, (self.n, 3)),)

    def project_all(self, inputs, dense=False):
        import torch
        q = torch.from_numpy(np.concatenate([i[0] for i in inputs])).cuda()
        out = self.tab.project(q, extra_flags=self.mode)
        return out[0], out[2], out[4]

    def pinned(self):
        import torch
        self.q_pin = torch.from_numpy(self.q_host).pin_memory().numpy()

    def host(self, out, dense=False):
        self.tab.project_host(self.q_pin, out=out[:4] + (None,), extra_flags=self.mode)

    def cpu_jobs(self, sample):
        sample = max(64, min(sample, 2048))
        desc = (f"first {sample} of the {self.n} queries, brute force over all "
                f"{self.num_segments} cubics of the {len(self.preps)} curves (per curve, min kept)")
        return [(_seg(p), self.q_host[:sample]) for p in self.preps], desc


class SurfaceWorkload:
    """cfg4: one prepared surface (64 x 64 net), the rank's 1e6 queries."""

    def __init__(self, cfg, rank, world, n_override):
        import torch
        from paper_2504_11498_b200 import prepare_surface
        from paper_2504_11498_b200.fixtures import random_surface
        c = CONFIGS[cfg]
        p = c["degree"]
        self.surface = random_surface(np.random.default_rng(0), p, p, 64, 64)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        self.prep = prepare_surface(self.surface)
        torch.cuda.synchronize()
        self.prep_ms = (time.perf_counter() - t0) * 1e3
        self.tab = self.prep.table
        self.n = n_override or c["n"]
        # the cell index is part of preparing a surface for dense batches
        t0 = time.perf_counter()
        self.tab._cell_flag(max(self.n, 1 << 20))
        torch.cuda.synchronize()
        self.cells_ms = (time.perf_counter() - t0) * 1e3
        self.n_total = world * self.n
        self.q_host = np.random.default_rng(1 + rank).uniform(0.0, 1.0, (self.n, 3))
        self.q = torch.from_numpy(self.q_host).cuda()
        self.num_segments = self.prep.num_patches
        self.h2d = self.n * 24
        self.p = p

    def step(self, counters=None, extra_flags=0, dense=False, sl=slice(None)):
        return self.tab.project(self.q[sl], counters=counters, extra_flags=extra_flags)

    def inputs(self, r, world):
        return (np.random.default_rng(1 + r).uniform(0.0, 1.0, (self.n, 3)),)

    def project_all(self, inputs, dense=False):
        import torch
        q = torch.from_numpy(np.concatenate([i[0] for i in inputs])).cuda()
        out = self.tab.project(q)
        return out[0], out[3], out[4]

    def pinned(self):
        import torch
        self.q_pin = torch.from_numpy(self.q_host).pin_memory().numpy()

    def host(self, out, dense=False):
        u, foot, dist, cand, seg = out
        # (u, v, foot, dist, patch): v rides in the int64 buffer's bytes
        self.tab.project_host(self.q_pin, out=(u, cand.view(np.float64), foot, dist, seg))

    def cpu_jobs(self, sample):
        sample = max(64, min(sample, 2048))
        desc = (f"first {sample} of the {self.n} queries, brute force over all "
                f"{self.num_segments} patches (mrep_surface_oracle.c)")
        return [("surface", (self.prep, self.q_host[:sample]))], desc


def run_reference(args, rank):
    if rank != 0:
        return
    if CONFIGS[args.config].get("nearest"):
        print(json.dumps({"impl": "reference", "unavailable": "the reference has no "
                          "nearest-over-set call (SPEC.md:497 non-goal); the mrep line's "
                          "cpu_baseline times the per-curve oracle instead"}), flush=True)
        return
    import oracle
    from oracle import prep as P
    cores = len(os.sched_getaffinity(0))
    if CONFIGS[args.config].get("surface"):
        from oracle import surface as OS
        from paper_2504_11498_b200.fixtures import random_surface
        pp = CONFIGS[args.config]["degree"]
        sf = random_surface(np.random.default_rng(0), pp, pp, 64, 64)
        pts, iv = OS.decompose(pp, pp, sf.knots_u.knots, sf.knots_v.knots, sf.control_points)
        sample = max(64, min(args.ref_sample // 16, 2048))
        q = np.random.default_rng(1).uniform(0.0, 1.0, (sample, 3))
        P = pts.reshape(-1, pp + 1, pp + 1, 3)
        I = iv.reshape(-1, 4)

        def run_one(qq):
            oracle.surface_project(P, I, pp, pp, qq, workers=cores)

        desc = (f"{sample} of the {args.config} queries per step, brute force over all {len(P)} "
                f"patches (mrep_surface_oracle.c: the reference has no surface code, this CPU "
                f"oracle defines the algorithm)")
        for _ in range(args.warmup):
            run_one(q[:32])
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            run_one(q)
            times.append(time.perf_counter() - t0)
        jobs = None
    elif args.config == "cfg3":
        from paper_2504_11498_b200.fixtures import mixed_curve_batch
        c = CONFIGS["cfg3"]
        curves = mixed_curve_batch(c["curves"])
        rng = np.random.default_rng(1)
        cid = (np.arange(c["n"]) % c["curves"]).astype(np.int32)
        rng.shuffle(cid)
        q_all = rng.uniform(0.0, 1.0, (c["n"], 3))
        stride = len(curves) // 50
        jobs, ns = [], 0
        for ci in range(0, len(curves), stride):
            cv = curves[ci]
            pr = P.prepare(cv.degree, np.array(cv.knots.knots), np.array(cv.control_points), 1e-4)
            jobs.append(((pr["seg_pts"], pr["seg_ta"], pr["seg_tb"], pr["seam_t"], pr["seam_pt"]),
                         q_all[cid == ci]))
            ns += len(pr["seg_ta"])
        sample = sum(len(j[1]) for j in jobs)
        desc = (f"{sample} queries of {len(jobs)} stratified curves (every {stride}th of "
                f"{len(curves)}, {ns} cubics, numpy restatement of prepare_curve), brute force "
                f"per curve")
    else:
        curve = make_curve(args.config)
        pr = P.prepare(*curve, 1e-4)
        seg = (pr["seg_pts"], pr["seg_ta"], pr["seg_tb"], pr["seam_t"], pr["seam_pt"])
        S = len(pr["seg_ta"])
        sample = args.ref_sample if args.config == "cfg2" else max(64, int(args.ref_sample * 510 / S))
        if CONFIGS[args.config]["queries"] == "on-curve":
            p_, k_, c_ = curve
            q = P.eval_curve(p_, k_, c_, np.random.default_rng(1).uniform(k_[0], k_[-1], sample))
        else:
            q = make_queries(args.config, 0, sample)
        jobs = [(seg, q)]
        desc = f"{sample} of the {args.config} queries per step, brute force over all {S} cubics"
    if jobs is not None:
        for _ in range(args.warmup):
            for seg, q in jobs:
                oracle.project_block(*seg, q[: max(100, len(q) // 10)], workers=cores)
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            for seg, q in jobs:
                oracle.project_block(*seg, q, workers=cores)
            times.append(time.perf_counter() - t0)
    ms = statistics.mean(times) * 1e3
    value = sample / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": CONFIGS[args.config]["scaling"],
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(args.config, CONFIGS[args.config]["n"]),
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": desc + (f", {cores} threads" if jobs is None else
                                               " (C restatement of _kernels._project_block, "
                                               f"bit-exact vs the reference), {cores} threads")},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mrep", choices=["mrep", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--n", "--queries-per-gpu", dest="n", type=int, default=0,
                    help="queries per GPU (default: the config's)")
    ap.add_argument("--ref-sample", type=int, default=131072)
    ap.add_argument("--cpu-sample", type=int, default=131072)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dense", action="store_true", help="brute-force kernel (reference semantics)")
    ap.add_argument("--verify-gather", action="store_true",
                    help="N > 1: rank 0 checks the gathered (t, distance, segment id) of the last "
                         "step bitwise against one projection of every rank's queries")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "mrep":
        # `python bench.py --gpus N` starts its own N ranks (one per GPU)
        sys.exit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    import torch
    import torch.distributed as dist
    ndev = torch.cuda.device_count()
    # one rank per GPU over NCCL; with fewer GPUs than ranks (the 1-GPU test
    # box) ranks share devices and gather over gloo -- flagged in config
    shared = world > ndev
    torch.cuda.set_device(local % ndev)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2504_11498_b200 import _lib as L

    cfg = CONFIGS[args.config]
    surf = CONFIGS[args.config].get("surface", False)
    wl = (CurveSetWorkload if args.config == "cfg3" else SurfaceWorkload if surf
          else NearestWorkload if cfg.get("nearest") else SingleCurve)(args.config, rank, world,
                                                                         args.n)
    n, n_total = wl.n, wl.n_total
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    counters = torch.zeros(L.NUM_COUNTERS, dtype=torch.int64, device="cuda")
    dense = args.dense and args.config != "cfg3"

    from paper_2504_11498_b200.sharding import gather_chunk, pack_results

    # N > 1: the step runs as CHUNKS query chunks; each chunk's (t, distance,
    # segment id) block is gathered to rank 0 asynchronously (NCCL's stream
    # waits for that chunk only) while the next chunk projects, so only the
    # last chunk's gather is exposed (overlap by chunking)
    chunks = 1 if world == 1 else CHUNKS
    bounds = [n * i // chunks for i in range(chunks + 1)]
    kmax = -(-(-(-n_total // world)) // chunks)
    # rank r's chunk i holds global queries [base_r + bounds[i], ...); the
    # gathered layout is chunk-major, unpermuted on rank 0 only when checked
    gathered = {}

    def run_step(counters=None, extra_flags=0):
        if chunks == 1:
            return wl.step(counters, extra_flags, dense=dense)
        works, outs = [], []
        for i in range(chunks):
            out = wl.step(counters, extra_flags, dense=dense, sl=slice(bounds[i], bounds[i + 1]))
            # surfaces (u, v, foot, dist, patch) -> (u, dist, patch)
            blk = (pack_results(out[0], out[3], out[4]) if surf
                   else pack_results(out[0], out[2], out[4]))
            if blk.shape[0] < kmax:  # uneven shards: pad to the common chunk size
                blk = torch.cat([blk, blk.new_zeros((kmax - blk.shape[0], 3))])
            w, bufs = gather_chunk(blk, world, rank, async_op=not shared)
            works.append(w)
            outs.append((out, bufs))
        for w in works:
            if w is not None:
                w.wait()  # the compute stream waits for the last gathers
        gathered["last"] = outs
        return outs[-1][0]

    # the clock sampler (an nvidia-smi child) starts before the warm-up, so its
    # start-up never lands inside a timed step
    clocks = ClockSampler(local)
    clocks.__enter__()
    # warm-up mirrors the timed loop exactly: the L2-flush fills (zero and
    # non-zero values take different paths) and the previous step's outputs
    # alive while the next step allocates (otherwise the allocator's first
    # second-buffer cudaMalloc lands in timed step 1 and stalls it)
    out = None
    for i in range(args.warmup):
        flush.fill_(float(i % 2))
        out = run_step()
    torch.cuda.synchronize()

    # ---- timed device steps (inputs resident in HBM) ----
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("bench_timed")  # ncu --nvtx-include bench_timed/
    for i in range(args.steps):
        flush.fill_(float(i))
        starts[i].record(stream)
        out = run_step()
        ends[i].record(stream)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    if world > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    gather_check = None
    if world > 1 and args.verify_gather and rank == 0:
        from paper_2504_11498_b200.sharding import unchunk
        outs = gathered["last"]
        got = unchunk([b for _, b in outs], world, n, bounds)
        ins = [wl.inputs(r, world) for r in range(world)]
        sizes = [len(i[0]) for i in ins]
        # rank r's rows: chunk blocks are kmax long; keep each chunk's real rows
        rows = []
        for r in range(world):
            br = [sizes[r] * i // chunks for i in range(chunks + 1)]
            for i in range(chunks):
                base = (r * chunks + i) * kmax
                rows.append(got[base: base + br[i + 1] - br[i]])
        got = torch.cat(rows).numpy()
        t_all, d_all, s_all = wl.project_all(ins, dense=dense)
        want = np.stack([t_all.cpu().numpy(), d_all.cpu().numpy(),
                         s_all.cpu().numpy().astype(np.float64)], 1)
        gather_check = {"queries": int(want.shape[0]),
                        "bitwise_equal": bool(got.shape == want.shape
                                              and np.array_equal(got, want))}
    ms = statistics.mean(step_ms)
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = n_total / (ms / 1e3)
    # own kernels per projection call (the timed steps' ncu launch lists,
    # profiles/r02_<cfg>_launch_shares.txt): ordering -- bucket sort (keys,
    # scan init, scan, scatter) from 2^16 queries, none below; cfg3: the
    # curve-rank counting sort (count, plan, scatter) -- then the wavefront:
    # traverse, pairs filter, pairs, clip, emit, unpermute (sorted batches),
    # fallback (surfaces: traverse, solve x2, filter, select x2, fallback);
    # dense mode: 2.  Per 2^23-query chunk.
    if args.config == "cfg3":
        sort_k = 3
    else:
        sort_k = 4 if min(n, 1 << 23) >= (1 << 16) else 0
    unperm = 1 if (sort_k and not surf and not dense) else 0
    launches_per_step = sort_k + (7 if surf else (6 + unperm if not dense else 2))
    launches_per_step *= max(1, -(-n // (1 << 23)))

    # ---- roofline: per-stage device times (CUDA events between the pipeline's
    #      kernels, recorded inside libmrep on this stream) x algorithmic work ----
    # work counters from one untimed step (the counting kernels' variant
    # adds atomics; the timed steps run without it)
    counters.zero_()
    wl.step(counters, dense=dense)
    c = counters.cpu().numpy().astype(np.float64)
    import ctypes
    reps = 7
    per_rep = []
    for _ in range(reps):
        flush.fill_(2.0)
        wl.step(extra_flags=L.MREP_TIMING, dense=dense)
        buf = (ctypes.c_double * 8)()
        L.lib().mrep_last_stage_times(buf, 8)
        per_rep.append(np.array(buf[:8]))
    stage = np.median(np.stack(per_rep), axis=0)  # robust to a one-off slow rep
    peak = ctypes.c_double()
    L.check(L.lib().mrep_fp64_peak(ctypes.byref(peak)))
    # pipeline time of one rank's projection (N > 1: the step also holds the
    # exposed tail of the gather, so take the library's stage sum instead)
    kms = statistics.mean(step_ms) if world == 1 else float(np.sum(stage))
    names = ["morton_sort", "traverse", "pairs", "clip", "select", "fallback"]
    work = {"traverse": F_BOX * c[L.CNT_BOXES] + F_SEAM * c[L.CNT_SEAMS],
            "pairs": F_PAIR * c[L.CNT_PAIRS], "clip": F_CLIP * c[L.CNT_SURVIVORS]}
    if surf:
        # per (query, patch) solve: (p+1)^2 seed evaluations + per Newton
        # iteration one jet and one line-search evaluation
        pp = wl.p
        f_s0 = 2 * 3 * (pp + 1) ** 2 + 12 * pp
        f_sj = 6 * 3 * (pp + 1) ** 2 + 40 * pp + 40
        names = ["morton_sort", "traverse", "solve", "clip", "select", "fallback"]
        work = {"traverse": F_BOX * c[L.CNT_BOXES] + 30.0 * c[L.CNT_SEAMS],
                "solve": c[L.CNT_PAIRS] * (pp + 1) ** 2 * f_s0
                + c[L.CNT_CLIP_ITERS] * (f_sj + f_s0)}
    stages = {}
    for i, nm in enumerate(names):
        ms_i = float(stage[i])
        ent = {"ms": ms_i}
        if nm in work and ms_i > 0:
            ent["tflops"] = work[nm] / (ms_i / 1e3) / 1e12
            ent["frac"] = ent["tflops"] / peak.value
        stages[nm] = ent
    flops = sum(work.values())
    dom = max((k for k in ("traverse", "pairs", "solve", "clip") if k in stages),
              key=lambda k: stages[k]["ms"]) if not dense else None
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof) and dom:
        try:
            pj = json.load(open(prof))
            per = pj.get("dram_bytes_per_launch_by_config", {}).get(args.config, {})
            base = f"surf_{dom}" if surf else f"wave_{dom}"
            traffic = per.get(base)
            if traffic is None:  # e.g. wave_traverse_group for a traverse stage
                traffic = next((v for k, v in sorted(per.items()) if k.startswith(base)), None)
            if traffic is None and args.config == pj.get("config", "cfg2"):
                traffic = pj.get("dram_bytes_per_launch", {}).get(f"wave_{dom}")
        except Exception:
            traffic = None
    achieved = stages[dom]["tflops"] if dom else flops / (kms / 1e3) / 1e12
    kname = (f"surf_{dom}" if surf else f"wave_{dom}") if dom else "project_kernel (dense)"
    roofline = {"bound": "fp64", "kernel": kname,
                "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s",
                "frac": achieved / peak.value, "traffic": traffic,
                "peak_source": "DFMA microbenchmark measured in this run (mrep_fp64_peak); "
                               "MEASURED_PEAKS.json has no FP64 figure",
                "flop_model": ("surface: (p+1)^2 seeds x (6(p+1)^2 + 12p) + Newton iterations x "
                               "(24(p+1)^2 + 52p + 40) per pair, 30/upper-bound point, 10/box "
                               "test (DESIGN.md 3b)" if surf else
                               "500/pair + 650/clipped survivor + 10/seam + 10/box test "
                               "(SURVEY.md 8(d); counts from the kernels' own counters)"),
                "stages": stages,
                "pipeline": {"ms": kms, "tflops": flops / (kms / 1e3) / 1e12,
                             "frac": flops / (kms / 1e3) / 1e12 / peak.value},
                "per_query": {"pairs": c[L.CNT_PAIRS] / n, "survivors": c[L.CNT_SURVIVORS] / n,
                              "seams": c[L.CNT_SEAMS] / n, "box_tests": c[L.CNT_BOXES] / n}}
    if dom == "traverse" and not surf:
        # the scan does little arithmetic: its roofline is the bytes it must
        # touch: 24 per query + 32 per box test (8-B list
        # entry + 24-B float box) + 24 per offered seam, against measured HBM
        # copy bandwidth (most of these bytes are L1/L2 hits; `traffic` is the
        # DRAM share from ncu)
        hbm = None
        try:
            hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
            hsrc = "MEASURED_PEAKS.json hbm_gbs (burst copy)"
        except Exception:
            hbm, hsrc = 7700.0, "B200_PROFILING.md fallback"
        tb = 24.0 * n + 32.0 * c[L.CNT_BOXES] + 24.0 * c[L.CNT_SEAMS]
        ach_gbs = tb / (stages["traverse"]["ms"] / 1e3) / 1e9
        roofline.update({"bound": "hbm", "achieved": ach_gbs, "peak": hbm, "unit": "GB/s",
                         "frac": ach_gbs / hbm, "peak_source": hsrc,
                         "bytes_model": "24/query + 32/box test + 24/offered seam "
                                        f"({tb / n:.0f} B per query)",
                         "fp64_view": {"achieved": achieved, "peak": peak.value,
                                       "unit": "TFLOP/s", "frac": achieved / peak.value}})
    if surf:
        roofline["per_query"] = {"patch_solves": c[L.CNT_PAIRS] / n,
                                 "newton_iters": c[L.CNT_CLIP_ITERS] / n,
                                 "bound_points": c[L.CNT_SEAMS] / n,
                                 "box_tests": c[L.CNT_BOXES] / n}
    elif args.config != "cfg3":
        roofline["dense_equivalent_tflops"] = ((F_PAIR * wl.num_segments
                                               + F_SEAM * (wl.num_segments + 1)) * n
                                               / (kms / 1e3) / 1e12)

    # ---- the reference's brute-force candidate count (MREP_CAND_EXACT, the
    #      Python API's default cand) on the FP64 tensor cores: one
    #      mma.sync m8n8k4 per 8 queries x 1 cubic, 64 flop per (query, cubic)
    #      pair; timed as its own stage (slot 6), not part of `value` ----
    if (isinstance(wl, SingleCurve) and not dense
            and wl.num_segments * n <= 2_000_000_000):
        dpk = ctypes.c_double()
        L.check(L.lib().mrep_dmma_peak(ctypes.byref(dpk)))
        counters.zero_()
        wl.step(counters, extra_flags=L.MREP_CAND_EXACT)
        unc = float(counters.cpu().numpy()[L.CNT_UNCERTAIN])
        cms = []
        for _ in range(reps):
            flush.fill_(3.0)
            wl.step(extra_flags=L.MREP_CAND_EXACT | L.MREP_TIMING)
            buf = (ctypes.c_double * 8)()
            L.lib().mrep_last_stage_times(buf, 8)
            cms.append(buf[6])
        cm = float(np.median(cms))
        tested = cand_pairs_tested(wl.tab, wl.q, wl.num_segments)
        ach = 64.0 * tested / (cm / 1e3) / 1e12
        roofline["cand_exact"] = {
            "kernel": ("cand_cells_kernel" if wl.tab.cand_cells is not None else
                       "cand_count_kernel") + " (mma.sync.m8n8k4.f64 sign screen + exact solve "
                      "of undecided pairs)", "bound": "tensor", "ms": cm, "achieved": ach,
            "peak": dpk.value, "unit": "TFLOP/s", "frac": ach / dpk.value,
            "peak_source": "DMMA m8n8k4 microbenchmark measured in this run (mrep_dmma_peak)",
            "flop_model": "64 FP64 tensor flop per (query, cubic) pair tested (8x8x4 MMA per 8 "
                          "queries); with the cand cell index a query tests only its cell's "
                          "uncertified cubics",
            "pairs_tested_per_query": tested / n,
            "dense_equivalent_tflops": 64.0 * wl.num_segments * n / (cm / 1e3) / 1e12,
            "uncertain_pairs_per_query": unc / n}

    # ---- e2e: host buffers through the C ABI (H2D + kernel + D2H per step) ----
    wl.pinned()
    outs = (torch.empty(n, dtype=torch.float64).pin_memory(),
            torch.empty((n, 3), dtype=torch.float64).pin_memory(),
            torch.empty(n, dtype=torch.float64).pin_memory(),
            torch.empty(n, dtype=torch.int64).pin_memory(),
            torch.empty(n, dtype=torch.int32).pin_memory())
    onp = tuple(o.numpy() for o in outs)
    for _ in range(2):
        wl.host(onp, dense=dense)
    e2e_times = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        wl.host(onp, dense=dense)
        e2e_times.append(time.perf_counter() - t0)
    clocks.__exit__(None, None, None)
    e2e_s = statistics.mean(e2e_times)
    if world > 1:
        tt = torch.tensor([e2e_s], dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    # the same host call returning the reference's own cand (MREP_CAND_EXACT,
    # the Python API's default): every output equal to the reference kernel's
    e2e_ref = None
    if (world == 1 and isinstance(wl, SingleCurve) and not dense
            and wl.num_segments * n <= 2_000_000_000):
        for _ in range(2):
            wl.host(onp, extra_flags=L.MREP_CAND_EXACT)
        ts_ref = []
        for _ in range(max(3, args.steps // 4)):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            wl.host(onp, extra_flags=L.MREP_CAND_EXACT)
            ts_ref.append(time.perf_counter() - t0)
        e2e_ref = {"value": n / statistics.mean(ts_ref), "unit": UNIT,
                   "h2d_bytes_per_step": wl.h2d, "d2h_bytes_per_step": n * 48,
                   "path": "mrep_project_host with MREP_CAND_EXACT: t, foot, distance and the "
                           "reference's brute-force cand (tensor-core pass + cand cell index)"}
    e2e = {"value": n_total / e2e_s, "unit": UNIT, "h2d_bytes_per_step": wl.h2d,
           # (t, foot, dist, cand) for curves; (u, v, foot, dist, patch) for surfaces
           "d2h_bytes_per_step": n * ((8 + 8 + 24 + 8 + 4) if surf else (8 + 24 + 8 + 8)),
           "path": ("mrep_project_batch_host" if args.config == "cfg3" else
                    "mrep_project_surface_host" if surf else "mrep_project_host")
           + " (C ABI, pinned host buffers, five-chunk pipeline on priority streams)"}

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cores = len(os.sched_getaffinity(0))
            jobs, desc = wl.cpu_jobs(args.cpu_sample)
            nq, dt = cpu_time(jobs, cores)
            nq /= getattr(wl, "cpu_div", 1)  # queries, not (query, curve) projections
            cpu = {"value": nq / dt, "unit": UNIT, "cores": cores, "kind": "port",
                   "sample": f"{desc} ({dt:.1f} s wall on {cores} threads); C restatement of "
                             f"_kernels._project_block, bit-exact vs the reference"}
        conf = dict(workload_config(args.config, n), parallelism=f"query-shard x{world}",
                    prep_ms=wl.prep_ms, cubics=wl.num_segments)
        prep_line = None
        if (world == 1 and not args.no_cpu_baseline and not surf
                and args.config in ("cfg2", "cfg3")):
            prep_line = prep_measure(wl, args.config)
        if world > 1:
            conf["gather"] = (f"(t, distance, segment id) to rank 0 in {chunks} chunks per step, "
                              + ("gloo through host memory (ranks share a GPU: a logic test, "
                                 "not a scaling number)" if shared else
                                 "NCCL, each chunk's gather overlapping the next chunk's projection"))
            if gather_check is not None:
                conf["gather_check"] = gather_check
        if getattr(wl, "cells_ms", None) is not None:
            if getattr(getattr(wl, "tab", None), "cells", None) is not None:
                conf["cell_index"] = {"build_ms": wl.cells_ms,
                                      "bytes": int(wl.tab.cells.numel() * 4)}
            elif getattr(wl, "cells_bytes", 0):
                conf["cell_index"] = {"build_ms": wl.cells_ms, "bytes": int(wl.cells_bytes),
                                      "kind": "one grid per curve (mrep_curveset_cells_build)"}
        sm_sorted = sorted(step_ms)
        conf["step_ms"] = {"median": statistics.median(step_ms), "min": sm_sorted[0],
                           "max": sm_sorted[-1], "argmax": int(np.argmax(step_ms))}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": cfg["scaling"], "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "config": conf,
                "e2e": e2e, "e2e_reference_cand": e2e_ref, "roofline": roofline,
                "cpu_baseline": cpu,
                "gpu_launches": launches_per_step * args.steps, "clocks": clocks.summary()}
        if prep_line is not None:
            line["preparation"] = prep_line
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
