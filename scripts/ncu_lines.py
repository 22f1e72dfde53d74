"""Aggregate an `ncu --page source --csv --print-source cuda,sass` dump by
CUDA source line: warp-stall samples, executed instructions, top stalls.

    python scripts/ncu_lines.py dump.csv [top] [inst]   (sort by instructions)"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur_file, cur_line, cur_src = "?", None, ""
agg = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0] != "":
        cur_line, cur_src = r[0], r[1]
        continue
    if r[2] in ("...", ""):
        continue
    key = (cur_file, cur_line)
    e = agg.setdefault(key, {"src": cur_src, "samples": 0, "inst": 0, "stalls": {}})
    try:
        e["samples"] += int(r[4])
        e["inst"] += int(r[7])
    except ValueError:
        continue
    for i, name in enumerate(hdr):
        if name.startswith("stall_") and "Not Issued" not in name:
            try:
                v = int(r[i])
            except ValueError:
                continue
            if v:
                e["stalls"][name] = e["stalls"].get(name, 0) + v
tot = sum(e["samples"] for e in agg.values()) or 1
order = "inst" if len(sys.argv) > 3 and sys.argv[3] == "inst" else "samples"
print(f"total instructions {sum(e['inst'] for e in agg.values())}")
for (f, ln), e in sorted(agg.items(), key=lambda kv: -kv[1][order])[:top]:
    st = sorted(e["stalls"].items(), key=lambda kv: -kv[1])[:3]
    st = " ".join(f"{k[6:]}={v}" for k, v in st)
    print(f"{100 * e['samples'] / tot:5.1f}% inst={e['inst']:>10d} {f}:{ln:<5} {e['src'].strip()[:70]:70s} {st}")
