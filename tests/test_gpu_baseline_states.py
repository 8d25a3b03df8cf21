"""Bit-exact parity on the BASELINE configurations' own states.

Each case builds the workload state exactly as bench.py does (bench.gpu_state: the host
RSA start of the configuration, grown on the device by srm_generate to its window), then
checks one device round against the CPU oracle on that full-size state:

  * grid: keys, sorted order and cell offsets (cell_grid.hpp:62-79, engine.hpp:144-166);
  * the round: accept decision and final position of every particle (the coloured
    Gauss-Seidel restatement of engine.hpp:89-107, oracle orc_sweep_round /
    orc_pl_sweep_round);
  * the reduction: overlap pairs and max penetration (orc_overlap_stats; platelets:
    orc_pl_pairs, every ordered pair of the reference's asymmetric test).

cfg4 is the bench's own window (10^7 spheres at f = 0.294); cfg2 is 10^6 spheres at
f = 0.392; cfg3 is 10^6 lognormal spheres in the L = 211.16 box grown from the clustered
start to f = 0.49 (crowded grid: the 4x4x4-brick near lists and the team sweep); cfg5 is 10^5
platelets of aspect ratio 100 from the recipe's rsa_platelets start (rho = 3.5).
The oracle is O(N) (binned pair search), about a minute at 10^7 on the host.
"""
import os
import sys

import numpy as np
import pytest

import orc
import paper_2605_18254_b200 as srm

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

pytestmark = pytest.mark.gpu


def _sphere_round_parity(ctx, cfg, c_m, dim):
    L = list(ctx.box[:dim])
    pos, r, ids = ctx.download()
    n = len(r)
    slot = np.arange(n, dtype=np.int32)
    cs = 2.5 * float(r.max()) + c_m
    keys, order, cell_start = ctx.grid_build(cs)
    k_o, dims, _ = orc.o_keys(dim, L, cs, pos)
    assert np.array_equal(keys, k_o), "cell keys differ from the oracle"
    o_order, o_cs = orc.o_sort(k_o, slot, int(np.prod(dims)))
    assert np.array_equal(order, o_order), "sorted order differs from the oracle"
    assert np.array_equal(cell_start, o_cs), "cell offsets differ from the oracle"
    del keys, order, cell_start, k_o, o_order, o_cs
    key, rid, it = srm.mix_seed(1234, 5), 3, 17
    st, acc = ctx.round(cs, c_m, bench.N_L, key, rid, it)
    p_d, r_d, id_d = ctx.download()
    xo, ao = orc.o_round(dim, L, pos, r, ids, slot, cs, c_m, bench.N_L, key, rid, it)
    assert np.array_equal(acc, ao), f"accept decisions differ ({int(np.sum(acc != ao))} of {n})"
    assert np.array_equal(p_d, xo), "positions differ from the oracle"
    assert np.array_equal(r_d, r) and np.array_equal(id_d, ids)
    o = orc.o_stats(dim, L, xo, r)
    assert st.overlap_pairs == o.overlap_pairs
    assert st.max_penetration == o.max_penetration
    return n, int(np.sum(ao != 255)), st


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4"])
def test_round_bit_exact_on_baseline_state(name):
    cfg = bench.CONFIGS[name]
    seed = srm.mix_seed(20260101, 0)
    ctx, c_m, prep = bench.gpu_state(srm, cfg, seed, 0)
    try:
        assert prep["f_window"] >= bench.F_WINDOW * cfg["f_target"] * (1 - 1e-12)  # the bench window
        n, movers, st = _sphere_round_parity(ctx, cfg, c_m, cfg["dim"])
        assert n == cfg["n"] and movers > 0.5 * n
        if name == "cfg3":  # crowded grid (> 1.8 per cell): the 4x4x4 bricks and the team sweep ran
            assert n > 1.8 * ctx.last_round_info()["cells"]
    finally:
        ctx.close()


def test_round_bit_exact_on_cfg5_platelets():
    cfg = bench.CONFIGS["cfg5"]
    seed = srm.mix_seed(20260101, 0)
    ctx, c_m, prep = bench.gpu_state(srm, cfg, seed, 0)
    try:
        L = [cfg["L"]] * 3
        pos, nrm, D, t, ids = ctx.download_platelets()
        n = len(D)
        assert n == cfg["n"] and np.allclose(D / t, cfg["aspect"])
        slot = np.arange(n, dtype=np.int32)
        rb = 0.5 * float((D + t).max())
        cs = 2.5 * rb + c_m
        key, rid, it = srm.mix_seed(99, 1), 2, 40
        ctx.set_rotation(cfg["c_r"])
        st, acc = ctx.round(cs, c_m, cfg["n_l"], key, rid, it)
        p_d, n_d, D_d, t_d, id_d = ctx.download_platelets()
    finally:
        ctx.close()
    xo, no, ao = orc.o_pl_round(L, pos, nrm, D, t, ids, slot, cs, c_m, cfg["c_r"], cfg["n_l"], key, rid, it)
    assert np.array_equal(acc, ao), f"accept decisions differ ({int(np.sum(acc != ao))} of {n})"
    assert np.array_equal(p_d, xo) and np.array_equal(n_d, no)
    assert np.array_equal(D_d, D) and np.array_equal(t_d, t) and np.array_equal(id_d, ids)
    assert st.overlap_pairs == orc.o_pl_pairs(L, xo, no, D, t, ids)
