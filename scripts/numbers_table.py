"""Markdown table of the bench lines in gpurun_out/bench_*.json."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = [("cfg1", "cfg1 (10⁴ on-curve, 61 cubics)"),
        ("cfg2", "**cfg2 (headline, 10⁶ onto 510 cubics)**"),
        ("cfg3", "cfg3 (10⁴ curves, 10⁶ queries)"),
        ("cfg4", "cfg4 (bicubic surface, 3721 patches)"),
        ("cfg4q", "cfg4q (biquintic surface, 3481 patches)"),
        ("cfg5", "cfg5 (10⁸ onto 10⁵ cubics)"),
        ("cfg6", "cfg6 (§8(f) nearest of 100 curves, 41k cubics)")]
ref = json.load(open(os.path.join(ROOT, "gpurun_out", "bench_ref.json")))
print("| Config | device pts/s | e2e pts/s | CPU port (16 thr) | e2e / CPU | dominant kernel, FP64 frac |")
print("|---|---|---|---|---|---|")
for c, name in rows:
    d = json.load(open(os.path.join(ROOT, "gpurun_out", f"bench_{c}.json")))
    cpu = ref["value"] if c == "cfg2" else d["cpu_baseline"]["value"]
    r = d["roofline"]
    print(f"| {name} | {d['value']:.3g} | {d['e2e']['value']:.3g} | {cpu:.3g}"
          f"{' (ref arm)' if c == 'cfg2' else ''} | {d['e2e']['value'] / cpu:,.0f}× | "
          f"`{r['kernel']}` {r['frac']:.3f} |")
