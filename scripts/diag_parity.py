"""Print GPU-vs-reference parity statistics for every golden fixture.

    python scripts/diag_parity.py

Not a test (tests/ assert the bars); this shows the raw mismatch picture.
"""
import glob
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2504_11498_b200 import _device as D  # noqa: E402

G = os.path.join(ROOT, "tests", "golden")


def ops():
    g = np.load(os.path.join(G, "quartic.npz"))
    r, c = D.quartic_roots(g["coeffs"])
    m = np.isfinite(g["roots"])
    print("quartic: count mismatch", int((c != g["counts"]).sum()), "of", len(c),
          "| root bit-mismatch", int((r[m] != g["roots"][m]).sum()), "of", int(m.sum()),
          "| max |dr|", float(np.nanmax(np.abs(r[m] - g["roots"][m]))) if m.any() else 0)
    nr, nc = D.newton_quartic_roots(g["coeffs"])
    m = np.isfinite(g["newton_roots"])
    print("newton: count mismatch", int((nc != g["newton_counts"]).sum()),
          "| root bit-mismatch", int((nr[m] != g["newton_roots"][m]).sum()))
    o = np.load(os.path.join(G, "ops.npz"))
    e = D.distance_poly(o["dp_P"], o["dp_q"])
    print("distance_poly 3d bit-mismatch", int((e != o["dp_e"]).sum()))
    e = D.distance_poly(o["dp_P2"], o["dp_q2"])
    print("distance_poly 2d bit-mismatch", int((e != o["dp_e2"]).sum()))
    R = D.restrict_ordinates(o["rs_b"], o["rs_lo"], o["rs_hi"])
    print("restrict bit-mismatch", int((R != o["rs_out"]).sum()))
    f, z = D.hull_cross(o["hull_b"])
    print("hull found mismatch", int((f != o["hull_found"].astype(bool)).sum()),
          "z mismatch", int((z != o["hull_z"]).sum()))
    bad = 0
    for it in (3, 8):
        sel = o["clip_iters"] == it
        for tol in (1e-9, 1e-6):
            s2 = sel & (o["clip_tol"] == tol)
            root, ok, used, w = D.clip_root(o["clip_b"][s2], tol, it)
            bad += int((root != o["clip_root"][s2]).sum() + (ok != o["clip_ok"][s2].astype(bool)).sum()
                       + (used != o["clip_used"][s2]).sum()
                       + (w != o["clip_widths"][s2][:, :it]).sum())
    print("clip_root mismatches", bad)
    ev = D.eval_ordinates(o["rs_b"], o["ev_u"])
    print("eval_ordinates bit-mismatch", int((ev != o["ev_out"]).sum()))
    pt = D.cubic_points(o["dp_P"], o["ev_u"])
    print("cubic_points bit-mismatch", int((pt != o["pt_out"]).sum()))
    b = D.rebase(o["dp_e"])
    T5 = o["T5"]
    print("rebase max dev vs T5@e", float(np.abs(b - o["dp_e"] @ T5.T).max()))


def projection():
    for f in sorted(glob.glob(os.path.join(G, "project_*.npz"))):
        z = np.load(f)
        args = (z["seg_pts"], z["seg_ta"], z["seg_tb"], z["seam_t"], z["seam_pt"])
        t, foot, dist, cand, stats, sound = D.project_block(
            *args, z["queries"], float(z["clip_tol"]), int(z["max_iter"]), int(z["soundness"]))
        rel = np.abs(dist - z["dist"]) / np.maximum(z["dist"], 1e-300)
        line = (f"{os.path.basename(f):28s} dense: t bit={np.mean(t == z['t']):.4f} "
                f"max|dt|={np.abs(t - z['t']).max():.2e} max rel dd={rel.max():.2e} "
                f"max|dd|={np.abs(dist - z['dist']).max():.2e} "
                f"cand eq={np.mean(cand == z['cand']):.4f} stats eq={np.mean((stats == z['stats']).all(1)):.4f}")
        tab = D.DeviceTable(*args)
        ts, fs, ds, cs, ss, _, _ = tab.project(z["queries"], float(z["clip_tol"]), int(z["max_iter"]))
        ts, ds = ts.cpu().numpy(), ds.cpu().numpy()
        line += (f" | screen: t==dense {np.mean(ts == t):.4f} dist==dense {np.mean(ds == dist):.4f}"
                 f" mean cand {cs.double().mean().item():.1f}")
        print(line)


def speed():
    import torch
    z = np.load(os.path.join(G, "project_cfg2.npz"))
    args = (z["seg_pts"], z["seg_ta"], z["seg_tb"], z["seam_t"], z["seam_pt"])
    tab = D.DeviceTable(*args)
    q = torch.rand((1_000_000, 3), dtype=torch.float64, device="cuda",
                   generator=torch.Generator(device="cuda").manual_seed(1))
    for screen, n in ((True, 1_000_000), (False, 100_000)):
        qq = q[:n].contiguous()
        tab.project(qq, screen=screen)
        torch.cuda.synchronize()
        cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
        t0 = time.perf_counter()
        tab.project(qq, screen=screen, counters=cnt)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        c = cnt.cpu().numpy()
        print(f"cfg2 screen={screen}: {n / dt / 1e6:.2f} M pts/s ({dt * 1e3:.1f} ms) "
              f"pairs/q={c[0] / n:.2f} surv/q={c[1] / n:.2f} clipit/surv={c[2] / max(c[1], 1):.2f} "
              f"seams/q={c[3] / n:.1f} boxes/q={c[4] / n:.1f} pass2={c[5]}")


if __name__ == "__main__":
    ops()
    projection()
    speed()
