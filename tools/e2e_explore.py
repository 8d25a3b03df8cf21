#!/usr/bin/env python
"""Exploration of full-size end-to-end growth for the crowded BASELINE configurations
(cfg3 polydisperse clustered, cfg5 platelets): runs srm_generate with live progress and
prints f every `every` iterations.  tools/e2e_explore.py cfg3|cfg5 [key=value ...]"""
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2605_18254_b200 as srm  # noqa: E402


def main():
    name = sys.argv[1]
    kw = dict(a.split("=") for a in sys.argv[2:])
    cfg = dict(bench.CONFIGS[name])
    n = int(float(kw.get("n", cfg["n"])))
    seed = int(kw.get("seed", 7))
    c_w = float(kw.get("c_w", cfg.get("c_w", bench.C_W)))
    n_k = int(kw.get("n_k", cfg.get("n_k", bench.N_K)))
    n_l = int(kw.get("n_l", cfg.get("n_l", bench.N_L)))
    iters = int(kw.get("iters", 1000))
    every = int(kw.get("every", 50))
    relax = int(kw.get("relax", 0))
    t0 = time.time()
    if cfg["kind"] == "poly":
        ncl = max(1, n // 1000)
        r_t = bench.poly_radii(n, seed)
        L = (np.sum(4.0 / 3.0 * math.pi * r_t ** 3) / cfg["f_target"]) ** (1.0 / 3.0)
        r0 = r_t * (cfg["f0"] / cfg["f_target"]) ** (1.0 / 3.0)
        pos, ids = srm.rsa_clustered(r0, [L] * 3, ncl, cfg["sigma"], 10000, seed)
        c_m = float(kw.get("c_m", cfg["cm_abs"]))
        ctx = srm.Context([L] * 3, n)
        ctx.upload(pos, r0, ids)
        c_r = 0.0
    else:
        Lb = cfg["L"] * (n / cfg["n"]) ** (1.0 / 3.0)
        L = Lb
        rho0 = float(kw.get("rho0", cfg["rho0"]))
        D0 = (rho0 * Lb ** 3 / n) ** (1.0 / 3.0)
        pos, nrm, ids = srm.rsa_platelets(n, D0, cfg["aspect"], [Lb] * 3, 100000, seed)
        ctx = srm.Context([Lb] * 3, n, shape="platelet")
        ctx.upload_platelets(pos, nrm, np.full(n, D0), np.full(n, D0 / cfg["aspect"]), ids)
        c_m = float(kw.get("c_m", cfg["cm_abs"]))
        c_r = float(kw.get("c_r", cfg["c_r"]))
        ctx.set_rotation(c_r)
    f0 = ctx.volume_fraction()
    print(f"{name} n={n} L={L:.3f} start f={f0:.5f} prep {time.time() - t0:.1f}s c_w={c_w} c_m={c_m} c_r={c_r} "
          f"n_k={n_k} n_l={n_l} relax={relax}", flush=True)
    if relax:
        rm = float(kw.get("relax_cm", c_m))
        t = time.time()
        ctx.relax_sweeps(rm, c_r, n_l, relax, srm.mix_seed(seed, 5))
        ctx.sync()
        print(f"  relax {relax} sweeps c_m={rm}: {time.time() - t:.2f}s", flush=True)
    last = [time.time()]

    def prog(r):
        if r.iteration % every == 0:
            now = time.time()
            print(f"  it {r.iteration} f={r.volume_fraction:.5f} acc={int(r.accepted)} t={r.elapsed_seconds:.2f}s "
                  f"(+{now - last[0]:.1f}s)", flush=True)
            last[0] = now

    p = srm.SrmParams(c_w=c_w, c_m=c_m, c_r=c_r, n_k=n_k, n_l=n_l, f_target=cfg["f_target"],
                      max_iterations=iters, seed=seed + 1, reorder_period=16)
    t = time.time()
    out = ctx.generate(p, 0, prog)
    ctx.sync()
    dt = time.time() - t
    st = ctx.overlap_stats(2.5 * ctx.max_bounding_radius())
    print(f"{name}: status {out.status} f={out.volume_fraction:.12f} iterations {out.iteration_count} "
          f"accepted {out.accepted_iterations} rounds {out.rounds}+{out.shake_rounds} shake, {dt:.1f}s, "
          f"overlaps {st.overlap_pairs}", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
