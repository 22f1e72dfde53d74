"""Small invocations of every device path, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python scripts/sanitize.py [stage ...]

Stages: prep (decompose + approximation + packing), curve (screened wavefront
in all traversal modes, cell index, dense kernel with stats), host (the
pipelined host-buffer C-ABI call), batch (curve set + scheduler), nearest,
surface (traversal, cell index, solve, filter, select), verify (GPU
oracle_project_batch).  Sizes are small: the sanitizers slow kernels 10-100x.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2504_11498_b200 import (  # noqa: E402
    _lib as L, BSplineCurve, prepare_curve, prepare_curve_set, project_batch, project_prepared,
    prepare_surface, project_surface_prepared, prepare_nearest_set, project_nearest)
from paper_2504_11498_b200.fixtures import (  # noqa: E402
    mixed_curve_batch, random_clamped_curve, random_surface)
from paper_2504_11498_b200.verify import oracle_project_batch  # noqa: E402

N = int(os.environ.get("SANITIZE_N", "2048"))


def curve(p=5, n=40):
    return random_clamped_curve(np.random.default_rng(0), p, n, 3, uniform_knots=True)


def stage_prep():
    prepare_curve(curve(7, 64))
    prepare_curve_set(mixed_curve_batch(8, max_control=96))


def stage_curve():
    prep = prepare_curve(curve())
    q = np.random.default_rng(1).uniform(0, 1, (N, 3))
    tab = prep.table
    qd = L.to_dev(q)
    for mode in (L.MREP_PACKET, L.MREP_PER_LANE, L.MREP_GROUP):
        tab.project(qd, extra_flags=mode)
    tab.CELL_MIN_QUERIES = 0  # instance override: build the cell index at this size
    tab.project(qd)
    project_prepared(prep, q, return_segments=True, return_spans=True)
    project_prepared(prep, q[:256], with_stats=True, soundness_samples=4)
    # exact cand: full tensor-core pass, then with the cand cell index
    tab.cand_tried = True
    tab.project(qd, extra_flags=L.MREP_CAND_EXACT)
    tab.build_cand_cells(8)
    tab.project(qd, extra_flags=L.MREP_CAND_EXACT | L.MREP_CAND_CELLS)


def stage_host():
    prep = prepare_curve(curve())
    q = np.random.default_rng(2).uniform(0, 1, (N, 3))
    prep.table.project_host(q)


def stage_batch():
    curves = mixed_curve_batch(12, max_control=128)
    cs = prepare_curve_set(curves)
    rng = np.random.default_rng(3)
    cid = rng.integers(0, len(curves), N).astype(np.int32)
    q = rng.uniform(0, 1, (N, 3))
    project_batch(cs, q, cid)
    for mode in (L.MREP_PACKET, L.MREP_PER_LANE, L.MREP_GROUP):
        cs.project_device(L.to_dev(q), L.to_dev(cid, torch.int32), extra_flags=mode)
    cs.project_host(q, cid)
    cs.build_cells(8)
    cs.project_device(L.to_dev(q), L.to_dev(cid, torch.int32))
    cs.free()


def stage_nearest():
    cs = prepare_curve_set(mixed_curve_batch(6, max_control=64))
    ns = prepare_nearest_set([cs[i] for i in range(6)])
    project_nearest(ns, np.random.default_rng(4).uniform(0, 1, (N, 3)))
    cs.free()


def stage_surface():
    sp = prepare_surface(random_surface(np.random.default_rng(5), 3, 3, 10, 10))
    q = np.random.default_rng(6).uniform(0, 1, (N, 3))
    project_surface_prepared(sp, q)
    tab = sp.table
    tab.CELL_MIN_QUERIES = 0
    tab.project(L.to_dev(q))
    tab.project_host(q)


def stage_verify():
    oracle_project_batch(curve(), np.random.default_rng(7).uniform(0, 1, (256, 3)), grid=512)


STAGES = {k[6:]: v for k, v in globals().items() if k.startswith("stage_")}

if __name__ == "__main__":
    torch.cuda.set_device(0)
    for name in (sys.argv[1:] or list(STAGES)):
        STAGES[name]()
        torch.cuda.synchronize()
        print("stage ok:", name, flush=True)
    # hand the caching allocator's blocks back so leak checks see only ours
    import gc
    gc.collect()
    torch.cuda.empty_cache()
