#!/usr/bin/env python
"""Profiling driver: prepare a bench workload state (scaled N allowed), then run a
few SRM rounds.  Used under ncu, e.g.

  ncu --set full -k regex:k_phase0 -s 2 -c 1 -o gpurun_out/prof python tools/profile_round.py --n 2000000
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2605_18254_b200 as srm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--n", type=int, default=0, help="particles (box scaled to keep the density)")
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--timing", action="store_true")
    ap.add_argument("--n_l", type=int, default=0, help="attempts per particle (default: the configuration's)")
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS[args.config])
    n = args.n or cfg["n"]
    box = (n / cfg["n"]) ** (1.0 / cfg["dim"])
    t0 = time.time()
    ctx, c_m, prep = bench.gpu_state(srm, cfg, 12345, 0, n=n, box=box)
    cs = 2.5 * ctx.max_bounding_radius() + c_m
    print("prep", prep, f"{time.time() - t0:.1f}s", flush=True)
    if args.timing:
        ctx.timing_enable(True)
    import ctypes
    rt = ctypes.CDLL("libcudart.so.12")
    ctx.sync()
    rt.cudaProfilerStart()  # ncu --profile-from-start off captures only the timed rounds
    ctx.stopwatch_start()
    st = ctx.rounds(cs, c_m, args.n_l or cfg.get("n_l", bench.N_L), 77, 0, 1, args.rounds)
    ms = ctx.stopwatch_stop()
    rt.cudaProfilerStop()
    print(f"{args.rounds} rounds: {ms:.3f} ms ({ms / args.rounds:.3f} ms/round), overlaps {st.overlap_pairs}, "
          f"movers {st.movers}", ctx.last_round_info(), flush=True)
    if args.timing:
        fam, calls = ctx.timing_get()
        print("family ms/round", [round(v / args.rounds, 4) for v in fam], calls)
    ctx.close()


if __name__ == "__main__":
    main()
