#!/usr/bin/env python
"""Per-source-line instruction and stall shares of one kernel in an ncu report:
tools/ncu_lines.py rep.ncu-rep [kernel-regex] [top]"""
import csv
import subprocess
import sys
from collections import defaultdict


def num(v):
    try:
        return int(v)
    except (TypeError, ValueError):
        return 0


def main(rep, kern=None, top=30):
    args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kern:
        args += ["--kernel-name", f"regex:{kern}"]
    rows = list(csv.reader(subprocess.run(args, capture_output=True, text=True).stdout.splitlines()))
    hdr = None
    inst, stall, text = defaultdict(int), defaultdict(int), {}
    cur = None
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        if r[0]:
            cur = int(r[0])
            text[cur] = r[1]
            continue
        d = dict(zip(hdr[2:], r[2:]))
        inst[cur] += num(d.get("Instructions Executed"))
        stall[cur] += num(d.get("Warp Stall Sampling (All Samples)"))
    ti, ts = sum(inst.values()) or 1, sum(stall.values()) or 1
    print(f"warp instructions {ti}, stall samples {ts}")
    for ln in sorted(inst, key=lambda k: -stall[k])[:top]:
        print(f"{ln:5d} inst {inst[ln] / ti:6.1%} stall {stall[ln] / ts:6.1%}  {text[ln].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None, int(sys.argv[3]) if len(sys.argv) > 3 else 30)
