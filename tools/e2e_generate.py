#!/usr/bin/env python
"""End-to-end time to f_target (SURVEY.md §8d protocol (ii)): the reference's own start
(rsa_place, bit-identical) grown by the device srm_generate to the configuration's full
f_target; prints iterations, rounds and device seconds.  tools/e2e_generate.py cfg2 [cfg4 ...]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2605_18254_b200 as srm  # noqa: E402


def main(names):
    for name in names:
        cfg = bench.CONFIGS[name]
        n, dim = cfg["n"], cfg["dim"]
        r0 = bench.radius_for(cfg["f0"], n, dim)
        rt = bench.radius_for(cfg["f_target"], n, dim)
        pos, ids = srm.rsa_place(np.full(n, r0), [1.0] * dim, srm.K_RSA_DEFAULT_ATTEMPTS, 7)
        with srm.Context([1.0] * dim, n) as ctx:
            ctx.upload(pos, np.full(n, r0), ids)
            p = srm.SrmParams(c_w=bench.C_W, c_m=cfg["cm_rel"] * rt, n_k=bench.N_K, n_l=bench.N_L,
                              f_target=cfg["f_target"], max_iterations=100000, seed=8, reorder_period=16)
            ctx.sync()
            t = time.time()
            out = ctx.generate(p)
            ctx.sync()
            dt = time.time() - t
            st = ctx.overlap_stats(2.5 * ctx.max_bounding_radius())
        print(f"{name}: N={n} f {cfg['f0']} -> {out.volume_fraction:.12f} in {out.iteration_count} iterations, "
              f"{out.rounds} growth + {out.shake_rounds} shake rounds, {dt:.3f} s, overlaps {st.overlap_pairs}",
              flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg2", "cfg4"])
