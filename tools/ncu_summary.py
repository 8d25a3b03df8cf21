#!/usr/bin/env python
"""Summarise an ncu report (one kernel): speed-of-light, occupancy, warp efficiency,
top SASS lines by stall samples and the opcode mix.  tools/ncu_summary.py rep.ncu-rep"""
import csv
import subprocess
import sys
from collections import Counter


def run(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout


def main(rep, top=25):
    rows = list(csv.reader(run(rep, "--page", "details").splitlines()))
    h = rows[0]
    keep = ("Duration", "Compute (SM) Throughput", "DRAM Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
            "Memory Throughput", "Achieved Occupancy", "Registers Per Thread", "Grid Size", "Block Size",
            "Avg. Active Threads Per Warp", "Issued Warp Per Scheduler", "Warp Cycles Per Issued Instruction",
            "Theoretical Occupancy")
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in keep:
            print(f"{d['Kernel Name'][:40]:40s} {d['Metric Name']:38s} {d['Metric Value']} {d['Metric Unit']}")
    raw = list(csv.reader(run(rep, "--page", "raw").splitlines()))
    for k, v in zip(raw[0], raw[2]):
        if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "smsp__inst_executed.sum",
                 "smsp__thread_inst_executed.sum"):
            print(f"{k:40s} {v} {raw[1][raw[0].index(k)]}")
    rows = list(csv.reader(run(rep, "--page", "source", "--print-source", "sass").splitlines()))
    h = rows[1]
    data = []
    for r in rows[2:]:
        if len(r) != len(h) or r[0] == "Address":
            break
        data.append(dict(zip(h, r)))
    S = "Warp Stall Sampling (All Samples)"
    I = "Instructions Executed"
    tot = sum(int(d[S] or 0) for d in data)
    print(f"stall samples {tot}, warp instructions {sum(int(d[I] or 0) for d in data)}")
    for d in sorted(data, key=lambda d: -int(d[S] or 0))[:top]:
        print(f"  {d['Address'][-5:]} {int(d[S] or 0) / max(tot, 1):6.1%} inst {d[I]:>10s} thr {d['Avg. Threads Executed']:>3s}  {d['Source'][:60]}")
    ops, st = Counter(), Counter()
    for d in data:
        t = d["Source"].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        ops[op] += int(d[I] or 0)
        st[op] += int(d[S] or 0)
    print("opcodes by instructions:", ops.most_common(16))
    print("opcodes by stalls:", st.most_common(10))


if __name__ == "__main__":
    main(sys.argv[1])
