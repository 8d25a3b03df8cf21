"""Thin circular platelets (SpherodiskShape) on the GPU: one round bit for bit against
the oracle's sweep (oracle/srm_oracle.c orc_pl_sweep_round, itself pinned to the
reference's overlap test in tests/test_oracle_platelets.py), the any-collision count,
and srm_generate to a target fraction with an all-pairs audit -- in the device-resident
graph and the host loop, which agree bit for bit on a budget-limited run."""
import math

import numpy as np
import pytest

import orc
import paper_2605_18254_b200 as srm

pytestmark = pytest.mark.gpu


def _state(n, L, seed, aspect=20.0):
    pos, nrm, ids = srm.rsa_platelets(n, 1.0, aspect, [L] * 3, 10000, seed)
    D = np.full(n, 1.0)
    return [L] * 3, pos, nrm, D, D / aspect, ids


@pytest.mark.parametrize("n,L,swell,c_m,c_r,n_l,seed", [(600, 6.0, 1.15, 0.05, 0.06, 8, 1),
                                                         (1500, 8.5, 1.25, 0.02, 0.02, 10, 2),
                                                         (450, 5.5, 1.0, 0.1, 0.2, 4, 3)])
def test_round_bit_exact_vs_oracle(n, L, swell, c_m, c_r, n_l, seed):
    Lb, pos, nrm, D, t, ids = _state(n, L, seed)
    D, t = D * swell, t * swell  # swollen: overlaps to resolve
    rb = 0.5 * (D.max() + t.max())
    cs = 2.5 * rb + c_m
    key, rid, it = 0xABCDEF1234 + seed, 2, 9
    with srm.Context(Lb, n, shape="platelet") as ctx:
        ctx.upload_platelets(pos, nrm, D, t, ids)
        ctx.set_rotation(c_r)
        st, acc = ctx.round(cs, c_m, n_l, key, rid, it)
        p_d, n_d, D_d, t_d, id_d = ctx.download_platelets()
    xo, no, ao = orc.o_pl_round(Lb, pos, nrm, D, t, ids, ids, cs, c_m, c_r, n_l, key, rid, it)
    assert np.array_equal(acc, ao)
    assert np.array_equal(p_d, xo) and np.array_equal(n_d, no)
    assert np.array_equal(D_d, D) and np.array_equal(t_d, t) and np.array_equal(id_d, ids)
    assert st.overlap_pairs == orc.o_pl_pairs(Lb, xo, no, D, t, ids)
    assert 0 < int(np.sum(ao != 255)) <= n


def test_round_bit_exact_rim_seed_fallback():
    """cfg 5's regime (aspect 100, rsa start at rho 3.5, swollen by c_w): about 1 pair
    in 4000 within reach leaves disks_within's 200 projections undecided (16 of the
    57803 start pairs here), and the team sweep resolves those with a rim seed per lane
    (k_sweep_pl_team); the round must still be the oracle's bit for bit."""
    n, aspect = 8000, 100.0
    L = 10.77 / 0.818  # cfg 5's number density in diameters
    pos, nrm, ids = srm.rsa_platelets(n, 1.0, aspect, [L] * 3, 100000, 5)
    D = np.full(n, 1.008)
    t = D / aspect
    cs = 2.5 * 0.5 * (D.max() + t.max()) + 0.01 / 0.818
    c_m, c_r, n_l, key = 0.01 / 0.818, 0.012, 10, 77
    with srm.Context([L] * 3, n, shape="platelet") as ctx:
        ctx.upload_platelets(pos, nrm, D, t, ids)
        ctx.set_rotation(c_r)
        st0 = ctx.overlap_stats(cs)  # k_overlap_pl: the same fallback, a seed per lane
        for rid in range(3):
            st, acc = ctx.round(cs, c_m, n_l, key, rid, 9)
        p_d, n_d, _, _, _ = ctx.download_platelets()
    x, nm = pos, nrm
    for rid in range(3):
        x, nm, ao = orc.o_pl_round([L] * 3, x, nm, D, t, ids, ids, cs, c_m, c_r, n_l, key, rid, 9)
    assert np.array_equal(acc, ao)
    assert np.array_equal(p_d, x) and np.array_equal(n_d, nm)
    assert st0.overlap_pairs == orc.o_pl_pairs([L] * 3, pos, nrm, D, t, ids) > 0
    assert st.overlap_pairs == orc.o_pl_pairs([L] * 3, x, nm, D, t, ids)


def test_overlap_stats_vs_oracle_and_reference():
    Lb, pos, nrm, D, t, ids = _state(600, 6.5, 4)
    for swell in (1.0, 1.3, 1.6):
        Dg, tg = D * swell, t * swell
        with srm.Context(Lb, len(D), shape="platelet") as ctx:
            ctx.upload_platelets(pos, nrm, Dg, tg, ids)
            st = ctx.overlap_stats(2.5 * 0.5 * (Dg.max() + tg.max()))
        want = orc.o_pl_pairs(Lb, pos, nrm, Dg, tg, ids)
        assert st.overlap_pairs == want
        anyc = orc.ref().ref_pl_any_collision(orc.P(orc.arr(Lb)), 2.5 * 0.5 * (Dg.max() + tg.max()), len(D),
                                              orc.P(pos), orc.P(nrm), orc.P(Dg), orc.P(tg), orc.P(ids))
        assert (st.overlap_pairs > 0) == bool(anyc)


def _generate(snap, p, device_loop):
    with srm.Context(snap.box, snap.n, shape="platelet") as ctx:
        ctx.upload_platelets(snap.pos, snap.normal, snap.diameter, snap.thickness, snap.id)
        ctx.set_generate_mode(device_loop)
        out = ctx.generate(p)
        return (out,) + ctx.download_platelets()


def test_generate_reaches_target_without_overlaps():
    Lb, pos, nrm, D, t, ids = _state(1000, 8.0, 5)
    snap = srm.PlateletSnapshot(Lb, pos, nrm, D * 0.9, t * 0.9, ids)
    snap.refresh_volume_fraction()
    ft = snap.volume_fraction * 1.6
    p = srm.SrmParams(c_w=0.02, c_m=0.02, c_r=0.03, n_k=10, n_l=10, f_target=ft, seed=11)
    res = srm.srm_generate(snap, p)
    assert res.status == srm.GenerateStatus.Converged
    assert abs(res.snapshot.volume_fraction / ft - 1.0) < 1e-12
    s = res.snapshot
    assert orc.o_pl_pairs(list(s.box), s.pos, s.normal, s.diameter, s.thickness, s.id) == 0
    assert np.allclose(np.linalg.norm(s.normal, axis=1), 1.0, atol=1e-12)


def test_device_loop_equals_host_loop_platelets():
    Lb, pos, nrm, D, t, ids = _state(700, 7.5, 6)
    snap = srm.PlateletSnapshot(Lb, pos, nrm, D, t, ids)
    snap.refresh_volume_fraction()
    p = srm.SrmParams(c_w=0.05, c_m=0.03, c_r=0.05, n_k=3, n_l=6, f_target=snap.volume_fraction * 3.0,
                      max_iterations=8, seed=13, reorder_period=3)
    a = _generate(snap, p, False)
    b = _generate(snap, p, True)
    assert a[0].status == b[0].status == 1
    for k in ("iteration_count", "accepted_iterations", "rounds", "shake_rounds"):
        assert getattr(a[0], k) == getattr(b[0], k), k
    assert a[0].volume_fraction == b[0].volume_fraction
    for x, y in zip(a[1:], b[1:]):
        assert np.array_equal(x, y)
