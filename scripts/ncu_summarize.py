"""Summarise ncu captures into profiles/ (JSON + text), run here (no GPU).

    python scripts/ncu_summarize.py <full.ncu-rep> <launches.csv|-> <tag> [config]

The per-kernel DRAM traffic goes into profiles/ncu_summary.json under
dram_bytes_per_launch_by_config[config] (bench.py reads it as `traffic`).
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "launch__registers_per_thread", "sm__warps_active.avg.per_cycle_active",
           "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__pcsamp_warps_issue_stalled_no_instructions",
           "smsp__pcsamp_warps_issue_stalled_wait",
           "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
           "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
           "smsp__pcsamp_warps_issue_stalled_branch_resolving",
           "launch__grid_size", "launch__block_size"]


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        ent = {"kernel": r[h.index("Kernel Name")]}
        for m in METRICS:
            if m in h:
                v = r[h.index(m)].replace(",", "")
                try:
                    ent[m] = float(v)
                except ValueError:
                    ent[m] = v
                ent[m + ".unit"] = units[h.index(m)]
        res.append(ent)
    return res


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    return [(r[ki], float(r[vi].replace(",", ""))) for r in rows[1:]]


def main():
    rep, ll, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    config = sys.argv[4] if len(sys.argv) > 4 else "cfg2"
    lst = launches(ll) if ll != "-" else []
    prof = os.path.join(ROOT, "profiles")
    if rep == "-":  # launch shares only
        return write_shares(prof, tag, lst)
    kern = full(rep)
    per = {}
    for k in kern:
        name = k["kernel"].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
        mult = 1e6 if k.get("dram__bytes_read.sum.unit") == "Mbyte" else (
            1e9 if k.get("dram__bytes_read.sum.unit") == "Gbyte" else 1e3
            if k.get("dram__bytes_read.sum.unit") == "Kbyte" else 1.0)
        # summed over the capture's launches of that kernel (one projection
        # call: per call, e.g. both surf_solve passes)
        per[name] = per.get(name, 0.0) + (k["dram__bytes_read.sum"] +
                                          k["dram__bytes_write.sum"]) * mult
    path = os.path.join(prof, "ncu_summary.json")
    summary = json.load(open(path)) if os.path.exists(path) else {}
    summary.setdefault("dram_bytes_per_launch_by_config", {})[config] = per
    summary.setdefault("kernels_by_config", {})[config] = kern
    summary.setdefault("sources", {})[config] = os.path.basename(rep)
    if config == "cfg2":
        summary.update({"tag": tag, "source": os.path.basename(rep),
                        "dram_bytes_per_launch": per, "kernels": kern})
    json.dump(summary, open(path, "w"), indent=1)
    with open(os.path.join(prof, f"{tag}_ncu_kernels.txt"), "w") as f:
        for k in kern:
            f.write(k["kernel"][:90] + "\n")
            for m in METRICS:
                if m in k:
                    f.write(f"    {m:62s} {k[m]} {k.get(m + '.unit', '')}\n")
    write_shares(prof, tag, lst)


def write_shares(prof, tag, lst):
    if not lst:
        return
    # launch list: share of device time per kernel name over the whole command
    tot = {}
    for name, ns in lst:
        key = name.split("(")[0][:80]
        tot[key] = tot.get(key, 0.0) + ns
    all_ns = sum(tot.values())
    with open(os.path.join(prof, f"{tag}_launch_shares.txt"), "w") as f:
        f.write(f"# {len(lst)} launches, ncu --metrics gpu__time_duration.sum "
                f"--clock-control none (cold, serialised)\n")
        for key, ns in sorted(tot.items(), key=lambda kv: -kv[1]):
            f.write(f"{100 * ns / all_ns:6.2f}%  {ns / 1e3:12.1f} us  {key}\n")
    print(open(os.path.join(prof, f"{tag}_launch_shares.txt")).read()[:2000])


if __name__ == "__main__":
    main()
