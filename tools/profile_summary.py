#!/usr/bin/env python
"""Turn a round's ncu outputs into the committed profiles/ summaries.

  tools/profile_summary.py TAG LAUNCHES.csv FULL.ncu-rep N_PARTICLES ROUNDS

LAUNCHES.csv: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--clock-control none --profile-from-start off --csv` over tools/profile_round.py (the
timed rounds only); FULL.ncu-rep: `ncu --set full` of the same command.  Writes
profiles/TAG_launches.md, profiles/TAG_full.md and profiles/TAG_traffic.json (DRAM
bytes per round of the migrate step = near lists + sweep, read by bench.py).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STEP = ("k_near_lists", "k_near_half", "k_near_tiles", "k_near_zero", "k_sweep_cells", "k_sweep_work", "k_sweep_queue",
        "k_sweep_pl_team",
        "k_sweep_warpq", "k_work_count", "k_work_scan", "k_work_scatter")
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0,
        "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    while rows and rows[0][0] != "ID":  # (the profiled program's own output precedes the table)
        rows.pop(0)
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    per = defaultdict(dict)
    for r in rows[1:]:
        v = float(r[ix["Metric Value"]].replace(",", "")) * UNIT.get(r[ix["Metric Unit"]], 1.0)
        per[(r[ix["ID"]], r[ix["Kernel Name"]].split("(")[0].replace("void ", ""))][r[ix["Metric Name"]]] = v
    return per


def full_table(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__grid_size", "launch__block_size"]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        try:  # global-load sectors per request (coalescing evidence)
            spr = f"{float(d['l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum']) / float(d['l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum']):.2f}"
        except (KeyError, ValueError, ZeroDivisionError):
            spr = ""
        res.append((d["ID"], d["Kernel Name"].split("(")[0].replace("void ", ""), [d.get(k, "") for k in keys] + [spr]))
    return keys, res, dict(zip(h, rows[1]))


def main(tag, lpath, rep, n, rounds):
    n, rounds = int(n), int(rounds)
    per = launches(lpath)
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for (_, name), m in per.items():
        a = agg[name]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0)
        a[3] += m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    lines = [f"# {tag}: ncu launch list, {rounds} SRM rounds, N = {n}",
             "", "Per-launch times are cold-cache and serialised (ncu), so compare SHARES, not absolutes.",
             "", "| kernel | launches | us / round | share | DRAM read MB / round | DRAM write MB / round | B / particle-round |",
             "|---|---|---|---|---|---|---|"]
    step_bytes = 0.0
    for name, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        rd, wr = a[2] / rounds, a[3] / rounds
        if name.split("<")[0].split("::")[-1] in STEP:
            step_bytes += rd + wr
        lines.append(f"| {name} | {a[0]} | {a[1] / rounds:.1f} | {a[1] / tot:.1%} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | "
                     f"{(rd + wr) / n:.1f} |")
    lines += ["", f"Total device time per round (serialised): {tot / rounds:.1f} us.",
              f"Migrate step (near lists + sweep) DRAM traffic: {step_bytes / 1e6:.1f} MB / round = "
              f"{step_bytes / n:.1f} B per particle-update (algorithmic: 56 B in 3D)."]
    open(os.path.join(ROOT, "profiles", f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    json.dump({"tag": tag, "n": n, "rounds": rounds, "step_kernels": list(STEP),
               "step_dram_bytes_per_round": step_bytes, "step_dram_bytes_per_update": step_bytes / n,
               "source": os.path.basename(lpath)},
              open(os.path.join(ROOT, "profiles", f"{tag}_traffic.json"), "w"), indent=1)
    if rep and os.path.exists(rep):
        keys, res, units = full_table(rep)
        short = ["time", "dram rd", "dram wr", "L2 hit %", "SM %", "mem %", "warps active %", "regs",
                 "threads/inst", "grid", "block", "ld sectors/req"]
        out = [f"# {tag}: ncu --set full (one launch per kernel, timed rounds)", "",
               "| id | kernel | " + " | ".join(short) + " |", "|" + "---|" * (len(short) + 2)]
        for i, name, v in res:
            out.append(f"| {i} | {name} | " + " | ".join(v) + " |")
        out += ["", "units: " + ", ".join(f"{s}={units.get(k, '')}" for s, k in zip(short, keys))]
        open(os.path.join(ROOT, "profiles", f"{tag}_full.md"), "w").write("\n".join(out) + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:6])
