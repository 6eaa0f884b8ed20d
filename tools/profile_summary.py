"""Summarise ncu captures of one sort into profiles/ (launch list with DRAM bytes per launch,
per-kind shares, key metrics of full captures) and profiles/traffic.json for bench.py.

    python tools/profile_summary.py --launches gpurun_out/launches_dram_H.csv --config H \
        --full gpurun_out/full_round_H.ncu-rep gpurun_out/full_base_H.ncu-rep --tag r01
"""
import argparse
import csv
import json
import os
import subprocess
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KIND = [("k_plan", "other"), ("k_epi", "other"), ("k_init", "other"), ("k_sample", "sample_splitters"), ("k_tree_from", "sample_splitters"), ("k_classify", "classify_flush"),
        ("k_prepare", "prepare"), ("k_moves", "empty_block_moves"), ("k_permute", "block_permute"),
        ("k_cleanup", "cleanup"), ("k_base", "base_case")]
FULL_KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
             "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
             "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
             "smsp__sass_branch_targets.sum", "smsp__sass_branch_targets_threads_divergent.sum",
             "smsp__sass_branch_targets_threads_uniform.sum", "smsp__thread_inst_executed.sum",
             "launch__registers_per_thread"]


def kind_of(name):
    for k, v in KIND:
        if k in name:
            return v
    return "other"


def read_launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    i_id, i_name, i_grid, i_blk = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Grid Size"), hdr.index("Block Size")
    i_m, i_v = hdr.index("Metric Name"), hdr.index("Metric Value")
    launches = OrderedDict()
    for r in rows[1:]:
        d = launches.setdefault(r[i_id], {"name": r[i_name], "grid": r[i_grid], "block": r[i_blk]})
        d[r[i_m]] = float(r[i_v].replace(",", ""))
    return list(launches.values())


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    res = []
    for r in rows[2:]:
        d = {"name": r[hdr.index("Kernel Name")]}
        for k in FULL_KEYS:
            if k in hdr:
                d[k] = r[hdr.index(k)]
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches", required=True)
    ap.add_argument("--config", default="H")
    ap.add_argument("--full", nargs="*", default=[])
    ap.add_argument("--tag", default="r01")
    a = ap.parse_args()
    L = read_launches(a.launches)
    tot = sum(l["gpu__time_duration.sum"] for l in L)
    kinds = OrderedDict()
    for l in L:
        k = kind_of(l["name"])
        d = kinds.setdefault(k, {"launches": 0, "ns": 0.0, "dram": 0.0})
        d["launches"] += 1
        d["ns"] += l["gpu__time_duration.sum"]
        d["dram"] += l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)
    lines = [f"# ncu summary, config {a.config} ({a.tag})", "",
             "One sort under `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
             "--clock-control none` (cold-cache, serialised launches: compare shares, not absolute times).", "",
             "| kind | launches | time (ms) | share | DRAM bytes / launch (GB) |", "|---|---|---|---|---|"]
    traffic = {}
    for k, d in kinds.items():
        per = d["dram"] / d["launches"]
        traffic[k] = per
        lines.append(f"| {k} | {d['launches']} | {d['ns'] / 1e6:.3f} | {d['ns'] / tot:.1%} | {per / 1e9:.3f} |")
    lines += ["", f"Total kernel time {tot / 1e6:.3f} ms.", "", "## Launches", "",
              "| kernel | grid | block | time (us) | DRAM read (MB) | DRAM write (MB) |", "|---|---|---|---|---|---|"]
    for l in L:
        nm = l["name"].split("(")[0].replace("void ", "")
        lines.append(f"| `{nm}` | {l['grid']} | {l['block']} | {l['gpu__time_duration.sum'] / 1e3:.1f} | "
                     f"{l.get('dram__bytes_read.sum', 0) / 1e6:.1f} | {l.get('dram__bytes_write.sum', 0) / 1e6:.1f} |")
    for rep in a.full:
        lines += ["", f"## Full capture `{os.path.basename(rep)}`", "",
                  "| kernel | " + " | ".join(k.split(".")[0] for k in FULL_KEYS) + " |",
                  "|---" * (len(FULL_KEYS) + 1) + "|"]
        for d in full_metrics(rep):
            nm = d["name"].split("(")[0].replace("void ", "")
            lines.append(f"| `{nm}` | " + " | ".join(str(d.get(k, "")) for k in FULL_KEYS) + " |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{a.tag}_ncu_summary_{a.config}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    allt = json.load(open(tp)) if os.path.exists(tp) else {}
    allt[a.config] = traffic
    json.dump(allt, open(tp, "w"), indent=1)
    print("\n".join(lines[:16]))


if __name__ == "__main__":
    main()
