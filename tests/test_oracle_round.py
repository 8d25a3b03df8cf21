"""Properties of the oracle's coloured Gauss-Seidel round -- CPU only.

* the cell-list search and the O(n^2) all-pairs search give identical rounds;
* the round never creates an overlap: after it, overlapping pairs are exactly the
  overlapping pairs among particles that did not move;
* rejected particles keep their exact bits (test_engine.cpp:65-86), movers move c_m;
* a lone particle moves exactly c_m on its first attempt (test_engine.cpp:53-63);
* c_m = 0 is the identity (test_engine.cpp:88-94);
* the colouring separates classes by more than any trial's reach.
"""
import numpy as np
import pytest

import orc


def _state(dim, n, f, seed, L=None):
    L = L or [1.0] * dim
    unit = np.pi if dim == 2 else 4.0 / 3.0 * np.pi
    r = (f * np.prod(L) / (n * unit)) ** (1.0 / dim)
    st, pos, ids, _ = orc.r_rsa(dim, L, np.full(n, r), 10000, seed)
    assert st == 0
    return L, pos, np.full(n, r), ids


@pytest.mark.parametrize("dim,n,f", [(2, 400, 0.45), (3, 400, 0.3), (2, 300, 0.6)])
def test_cells_equal_brute(dim, n, f):
    L, pos, r, ids = _state(dim, n, min(f, 0.5 if dim == 2 else 0.3), 3)
    r = r * (f / min(f, 0.5 if dim == 2 else 0.3)) ** (1 / dim)  # swell: some overlaps
    c_m = 0.2 * r[0]
    cs = 2.5 * r.max() + c_m
    a = orc.o_round(dim, L, pos, r, ids, ids, cs, c_m, 8, 99, 2, 5, brute=False)
    b = orc.o_round(dim, L, pos, r, ids, ids, cs, c_m, 8, 99, 2, 5, brute=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("dim,f,swell", [(2, 0.5, 1.02), (3, 0.3, 1.02), (2, 0.7, 1.0), (3, 0.35, 1.05)])
def test_round_never_creates_overlap(dim, f, swell):
    L, pos, r, ids = _state(dim, 600, min(f, 0.45 if dim == 2 else 0.3), 11)
    r = r * (f / min(f, 0.45 if dim == 2 else 0.3)) ** (1 / dim) * swell
    c_m = 0.1 * r[0]
    xnew, acc = orc.o_round(dim, L, pos, r, ids, ids, 2.5 * r.max() / swell + c_m, c_m, 10, 1234, 0, 1)
    moved = acc != 255
    assert moved.sum() > 0
    # non-movers keep their exact bits, movers moved exactly one proposal
    assert np.array_equal(xnew[~moved], pos[~moved])
    # overlapping pairs after the round == overlapping pairs among non-movers
    after = orc.o_stats(dim, L, xnew, r)
    stay = np.where(~moved)[0]
    among = orc.o_stats(dim, L, pos[stay], r[stay], ids[stay]) if len(stay) > 1 else None
    assert after.overlap_pairs == (among.overlap_pairs if among else 0)
    if among:
        assert after.max_penetration == among.max_penetration


def test_caged_particle_reverts_bit_exactly():
    # hexagonal cage at near contact (test_engine.cpp:65-86): whatever the sweep order,
    # a particle that rejects keeps its exact bits and a mover moved exactly one trial
    pos = [[0.5, 0.5]] + [[0.5 + 0.2000000001 * np.cos(k * np.pi / 3), 0.5 + 0.2000000001 * np.sin(k * np.pi / 3)]
                          for k in range(6)]
    pos = orc.arr(pos)
    r = np.full(7, 0.1)
    ids = np.arange(7, dtype=np.int32)
    for n_l in (1, 16):
        xnew, acc = orc.o_round(2, [1.0, 1.0], pos, r, ids, ids, 0.25, 0.05, n_l, 99, 0, 0)
        for i in range(7):
            if acc[i] == 255:
                assert np.array_equal(xnew[i], pos[i])
            else:
                assert np.linalg.norm(xnew[i] - pos[i]) == pytest.approx(0.05, rel=1e-12)


def test_single_particle_moves_c_m():
    pos = orc.arr([[0.5, 0.5]])
    xnew, acc = orc.o_round(2, [1.0, 1.0], pos, orc.arr([0.1]), [0], [0], 0.25, 0.05, 4, 17, 0, 0)
    assert acc[0] == 0
    assert np.linalg.norm(xnew[0] - pos[0]) == pytest.approx(0.05, rel=1e-12)


def test_zero_step_is_identity():
    L, pos, r, ids = _state(2, 100, 0.2, 5)
    xnew, acc = orc.o_round(2, L, pos, r, ids, ids, 2.5 * r.max(), 0.0, 4, 1, 0, 0)
    assert np.array_equal(xnew, pos)


def test_round_depends_on_key_not_on_storage_order():
    # the parallel round is a function of (state, slot), not of the array order
    L, pos, r, ids = _state(3, 500, 0.3, 8)
    r = r * 1.03
    c_m = 0.1 * r[0]
    cs = 2.5 * r.max() + c_m
    a_x, a_acc = orc.o_round(3, L, pos, r, ids, ids, cs, c_m, 6, 77, 1, 3)
    perm = np.random.default_rng(0).permutation(len(r))
    b_x, b_acc = orc.o_round(3, L, pos[perm], r[perm], ids[perm], ids[perm], cs, c_m, 6, 77, 1, 3)
    assert np.array_equal(b_x, a_x[perm]) and np.array_equal(b_acc, a_acc[perm])


@pytest.mark.parametrize("dim,L,cs,maxr,c_m", [(3, [1, 1, 1], 0.05, 0.018, 0.005), (3, [1, 1, 1], 0.07, 0.02, 0.02),
                                               (2, [1.0, 0.3], 0.02, 0.007, 0.001), (3, [0.2, 1, 1], 0.05, 0.015, 0.01)])
def test_colouring_separates_classes(dim, L, cs, maxr, c_m):
    dims, edge = orc.o_grid(dim, L, cs)
    m, ncol = orc.o_colouring(dim, L, cs, maxr, c_m)
    reach = 2 * maxr + 3 * c_m
    for a in range(dim):
        n = dims[a]
        body = m[a] * (n // m[a])
        col = [x % m[a] if x < body else m[a] + x - body for x in range(n)]
        assert max(col) + 1 == ncol[a]
        # same-colour coordinates are farther apart (cyclically) than the reach,
        # unless the axis is whole (every coordinate its own colour)
        for x in range(n):
            for y in range(n):
                if x != y and col[x] == col[y]:
                    gap = min(abs(x - y), n - abs(x - y)) - 1
                    assert gap * edge[a] >= reach
