"""The oracle's platelet restatement (oracle/srm_oracle.c: disks_within, spherodisk
overlap, measure, rotation) pinned against the reference itself (oracle/_ref: the
unmodified spherodisk.hpp / spherodisk.cpp) and against the known answers of the
reference's test_platelets.cpp."""
import math

import numpy as np
import pytest

import orc


def unit(v):
    v = np.asarray(v, float)
    return v / np.linalg.norm(v)


def test_known_answers_test_platelets_cpp():
    # test_platelets.cpp:60-82 (distances), via disks_within at thresholds around them
    ez, ex = [0.0, 0.0, 1.0], [1.0, 0.0, 0.0]
    o = orc.orc()
    P, a = orc.P, orc.arr
    for c2, n2, want in (([0, 0, 0.3], ez, 0.3), ([1.4, 0, 0], ez, 0.4), ([0, 0, 0], ex, 0.0),
                         ([1.3, 0, 0.2], ez, math.sqrt(0.2 ** 2 + (1.3 - 1.0) ** 2))):
        got = orc.ref().ref_pl_disk_distance(P(a([0, 0, 0])), P(a(ez)), 0.5, P(a(c2)), P(a(n2)), 0.5)
        assert got == pytest.approx(want, abs=1e-9)
        for thr in (want * 0.999 - 1e-12, want * 1.001 + 1e-12):
            mine = o.orc_pl_disks_within(P(a([0, 0, 0])), P(a(ez)), 0.5, P(a(c2)), P(a(n2)), 0.5, thr)
            theirs = orc.ref().ref_pl_disks_within(P(a([0, 0, 0])), P(a(ez)), 0.5, P(a(c2)), P(a(n2)), 0.5, thr)
            assert int(mine) == theirs == int(want <= thr)
    # test_platelets.cpp: coaxial parallel at centre separation exactly t -> overlap (inclusive)
    L = [10.0, 10.0, 10.0]
    assert orc.o_pl_overlap(L, [5, 5, 5], ez, 1.0, 0.1, [5, 5, 5.1], ez, 1.0, 0.1) == 1
    assert orc.r_pl_overlap(L, [5, 5, 5], ez, 1.0, 0.1, [5, 5, 5.1], ez, 1.0, 0.1) == 1


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_overlap_matches_reference_on_random_pairs(seed):
    rng = np.random.default_rng(seed)
    L = [4.0, 4.0, 4.0]
    n_pairs, hits = 3000, 0
    for _ in range(n_pairs):
        D1, D2 = rng.uniform(0.3, 1.0, 2)
        t1, t2 = D1 / rng.uniform(5, 150), D2 / rng.uniform(5, 150)
        pa = rng.uniform(0, 4, 3)
        # near contact most of the time: separation around the sum of the bounding radii
        sep = rng.uniform(0.0, 0.6 * (D1 + D2 + t1 + t2))
        pb = np.mod(pa + unit(rng.normal(size=3)) * sep, 4.0)
        na, nb = unit(rng.normal(size=3)), unit(rng.normal(size=3))
        if rng.uniform() < 0.2:  # near-parallel plates: the slow-convergence regime
            nb = unit(na + 1e-6 * rng.normal(size=3))
        for args in ((pa, na, D1, t1, pb, nb, D2, t2), (pb, nb, D2, t2, pa, na, D1, t1)):
            mine = orc.o_pl_overlap(L, *args)
            theirs = orc.r_pl_overlap(L, *args)
            assert mine == theirs, args
            hits += mine
    assert 0.1 * n_pairs < hits < 1.9 * n_pairs  # both outcomes well represented


def test_measure_and_rotation_match_reference():
    rng = np.random.default_rng(5)
    for _ in range(200):
        D = rng.uniform(0.01, 2.0)
        t = D / rng.uniform(1.0, 200.0)
        assert orc.orc().orc_pl_measure(D, t) == orc.ref().ref_pl_measure(D, t)
    # rotation: the oracle's propose formula vs rotate_about_axis with the same angle
    for _ in range(200):
        v, axis = unit(rng.normal(size=3)), unit(rng.normal(size=3))
        ang = rng.uniform(0, 0.5)
        out = np.zeros(3)
        orc.ref().ref_pl_rotate(orc.P(orc.arr(v)), orc.P(orc.arr(axis)), ang, orc.P(out))
        c, s = math.cos(ang), math.sin(ang)
        cr = np.array([axis[1] * v[2] - axis[2] * v[1], axis[2] * v[0] - axis[0] * v[2], axis[0] * v[1] - axis[1] * v[0]])
        dv = 0.0
        for k in range(3):
            dv += axis[k] * v[k]
        mine = np.array([(v[k] * c + cr[k] * s) + axis[k] * (dv * (1.0 - c)) for k in range(3)])
        assert np.array_equal(mine, out)


def test_pair_count_agrees_with_reference_any_collision():
    st, pos, nrm, ids = orc.r_rsa_platelets(300, 1.0, 20.0, [6.0, 6.0, 6.0], 10000, 4)
    assert st == 0
    D = np.full(300, 1.0)
    t = D / 20.0
    L = [6.0, 6.0, 6.0]
    assert orc.o_pl_pairs(L, pos, nrm, D, t, ids) == 0  # RSA: no contacts
    assert orc.ref().ref_pl_any_collision(orc.P(orc.arr(L)), 2.5 * 0.525, 300, orc.P(pos), orc.P(nrm), orc.P(D),
                                          orc.P(t), orc.P(ids)) == 0
    Dg, tg = D * 1.6, t * 1.6  # swollen: collisions appear
    pairs = orc.o_pl_pairs(L, pos, nrm, Dg, tg, ids)
    anyc = orc.ref().ref_pl_any_collision(orc.P(orc.arr(L)), 2.5 * 0.84, 300, orc.P(pos), orc.P(nrm), orc.P(Dg),
                                          orc.P(tg), orc.P(ids))
    assert pairs > 0 and anyc == 1


@pytest.mark.parametrize("seed,n,L", [(1, 400, 6.0), (7, 650, 6.5)])
def test_product_rsa_platelets_is_the_reference(seed, n, L):
    import paper_2605_18254_b200 as srm
    pos, nrm, ids = srm.rsa_platelets(n, 1.0, 20.0, [L] * 3, 10000, seed)
    st, p2, n2, i2 = orc.r_rsa_platelets(n, 1.0, 20.0, [L] * 3, 10000, seed)
    assert st == 0
    assert np.array_equal(pos, p2) and np.array_equal(nrm, n2) and np.array_equal(ids, i2)
