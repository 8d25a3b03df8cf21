"""Small SRM rounds through every kernel family, for compute-sanitizer.

  compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_rounds.py

Covers: the grid rebuild (k_keys, k_scan_lookback with several look-back tiles,
k_scatter, k_cellsort, k_gather), the near lists (k_near_tiles sparse bricks, the
crowded 4x4x4 bricks with the overflow pool, the global k_near_lists), every sweep
kernel (k_sweep_warpq, k_sweep_trials, k_sweep_team, k_sweep_pl_team; forced through
SRM_B200_SWEEP), the reductions (k_stats_sweep, k_overlap_pl, k_reduce_*), the device
RSA and the device-resident generate graph.  Sizes are small (sanitizers slow kernels
down 10-100x) but large enough that every brick / tile / look-back path is taken.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_18254_b200 as srm  # noqa: E402


def sphere_state(dim, n, f, seed, poly=False):
    L = [1.0] * dim
    unit = np.pi if dim == 2 else 4.0 / 3.0 * np.pi
    if poly:
        rng = np.random.default_rng(seed)
        rel = np.clip(rng.lognormal(-0.02, 0.2, n), 0.5, 2.0)
        r = rel * (f / (unit * np.sum(rel ** dim))) ** (1.0 / dim)
    else:
        r = np.full(n, (f / (n * unit)) ** (1.0 / dim))
    pos, ids = srm.rsa_place(r, L, 10000, seed)
    return L, pos, r, ids


def rounds(L, pos, r, ids, swell, cm_rel, tag):
    r = r * swell
    c_m = cm_rel * r.max()
    cs = 2.5 * r.max() / swell + c_m
    with srm.Context(L, len(r)) as ctx:
        ctx.upload(pos, r, ids)
        for k in range(2):
            st, _ = ctx.round(cs, c_m, 6, 0x5EED + k, k, 1, with_candidates=(k == 0))
        ctx.overlap_stats(cs)
        ctx.volume_fraction()
        info = ctx.last_round_info()
    print(f"{tag}: overlaps {st.overlap_pairs} movers {st.movers} cells {info['cells']}", flush=True)


def main():
    kernels = ["", "lane", "trials", "team"]
    for kern in kernels:
        if kern:
            os.environ["SRM_B200_SWEEP"] = kern
        else:
            os.environ.pop("SRM_B200_SWEEP", None)
        rounds(*sphere_state(3, 12000, 0.25, 1), 1.03, 0.05, f"3D sparse bricks [{kern or 'auto'}]")
        rounds(*sphere_state(3, 6000, 0.12, 2, poly=True), 1.05, 0.6, f"3D poly crowded [{kern or 'auto'}]")
        rounds(*sphere_state(2, 4000, 0.4, 3), 1.02, 0.1, f"2D global lists [{kern or 'auto'}]")
    os.environ.pop("SRM_B200_SWEEP", None)
    # platelets: team sweep + k_overlap_pl
    n, aspect, L = 1200, 20.0, 9.0
    pos, nrm, ids = srm.rsa_platelets(n, 1.0, aspect, [L] * 3, 10000, 4)
    D = np.full(n, 1.2)
    with srm.Context([L] * 3, n, shape="platelet") as ctx:
        ctx.upload_platelets(pos, nrm, D, D / aspect, ids)
        ctx.set_rotation(0.05)
        st, _ = ctx.round(2.5 * 0.5 * 1.2 * (1 + 1 / aspect) + 0.05, 0.05, 6, 7, 0, 1)
    print(f"platelets: overlaps {st.overlap_pairs}", flush=True)
    # device RSA, device-resident generate graph (host loop too)
    with srm.Context([1.0] * 3, 3000) as ctx:
        r0 = np.full(3000, (0.1 * 3 / (4 * np.pi * 3000)) ** (1 / 3))
        ctx.rsa_device(r0, 11)
        out = ctx.generate(srm.SrmParams(c_w=0.05, c_m=0.1 * r0[0], f_target=0.2, seed=3, reorder_period=2))
        ctx.set_generate_mode(False)
        out2 = ctx.generate(srm.SrmParams(c_w=0.05, c_m=0.1 * r0[0], f_target=0.25, seed=3))
    print(f"generate: f {out.volume_fraction:.4f} -> {out2.volume_fraction:.4f}", flush=True)
    print("sanitize_rounds: done", flush=True)


if __name__ == "__main__":
    main()
