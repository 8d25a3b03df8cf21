#!/usr/bin/env python
"""End-to-end time to f_target at the BASELINE sizes (SURVEY.md §8d protocol (ii)).

Each configuration starts from its bench start (bench.py CONFIGS: cfg1 uniform centres
with r0 = half the smallest centre distance; cfg2 / cfg4 reference rsa_place at
f0 = 0.1; cfg3 the clustered start; cfg5 the recipe's rsa_platelets at rho 3.5) and is
grown by the device srm_generate to the FULL f_target with the configuration's
end-to-end protocol (bench.E2E_PARAMS).  Prints iterations, rounds, device seconds and
the zero-overlap audit.  --reference also times the reference engine (oracle/_ref, one
host core) on the same start where it finishes in minutes (cfg1).

  tools/e2e_generate.py [cfg1 cfg2 ...] [--reference]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import bench  # noqa: E402
import paper_2605_18254_b200 as srm  # noqa: E402


def main(names, reference):
    for name in names:
        cfg = dict(bench.CONFIGS[name])
        seed = 7
        t0 = time.time()
        ctx, c_m, params, start = bench.e2e_start(srm, cfg, seed, 0)
        prep = time.time() - t0
        ctx.sync()
        t = time.time()
        out = ctx.generate(params)
        ctx.sync()
        dt = time.time() - t
        if cfg["kind"] == "platelet":
            st = ctx.overlap_stats(2.5 * ctx.max_bounding_radius())
        else:
            st = ctx.overlap_stats(2.5 * ctx.max_bounding_radius())
        print(f"{name}: N={cfg['n']} f {start['f0']:.4g} -> {out.volume_fraction:.12f} (target {cfg['f_target']}) "
              f"status {out.status} in {out.iteration_count} iterations ({out.accepted_iterations} accepted), "
              f"{out.rounds} growth + {out.shake_rounds} shake rounds, {dt:.3f} s device loop "
              f"(start prep {prep:.1f} s), overlaps {st.overlap_pairs}; protocol c_w={params.c_w} c_m={params.c_m:.4g} "
              f"n_k={params.n_k} n_l={params.n_l}", flush=True)
        if reference and name == "cfg1":
            import orc
            pos, r, ids = start["pos"], start["radius"], start["ids"]
            tr = time.time()
            stt, _, _, _, it, f, acc = orc.r_generate(2, [1.0, 1.0], pos, r, ids, params.c_w, params.c_m, params.n_k,
                                                      params.n_l, params.f_target, params.max_iterations, params.seed, 16)
            print(f"{name} reference (1 core): status {stt} f={f:.12f} in {it} iterations, {time.time() - tr:.2f} s",
                  flush=True)
        ctx.close()


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    main(args or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"], "--reference" in sys.argv)
