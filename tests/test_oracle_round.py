"""Properties of the oracle's parallel round -- CPU only.

* the cell-list search and the O(n^2) all-pairs search give identical rounds;
* the round never creates an overlap: after it, overlapping pairs are exactly the
  overlapping pairs among particles that did not move;
* a caged particle reverts bit-exactly (test_engine.cpp:65-86);
* a lone particle moves exactly c_m on its first attempt (test_engine.cpp:53-63);
* c_m = 0 is the identity (test_engine.cpp:88-94).
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
    a = orc.o_round(dim, L, pos, r, ids, ids, c_m, 8, 99, 2, 5, brute=False)
    b = orc.o_round(dim, L, pos, r, ids, ids, c_m, 8, 99, 2, 5, brute=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("dim,f,swell", [(2, 0.5, 1.02), (3, 0.3, 1.02), (2, 0.7, 1.0), (3, 0.35, 1.05)])
def test_round_never_creates_overlap(dim, f, swell):
    L, pos, r, ids = _state(dim, 600, min(f, 0.45 if dim == 2 else 0.3), 11)
    r = r * (f / min(f, 0.45 if dim == 2 else 0.3)) ** (1 / dim) * swell
    c_m = 0.1 * r[0]
    xnew, acc = orc.o_round(dim, L, pos, r, ids, ids, c_m, 10, 1234, 0, 1)
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
    # hexagonal cage at near contact (test_engine.cpp:65-86)
    pos = [[0.5, 0.5]] + [[0.5 + 0.2000000001 * np.cos(k * np.pi / 3), 0.5 + 0.2000000001 * np.sin(k * np.pi / 3)]
                          for k in range(6)]
    pos = orc.arr(pos)
    r = np.full(7, 0.1)
    ids = np.arange(7, dtype=np.int32)
    # In the parallel round the cage itself moves from phase 1 on (in the reference,
    # particle 0 is swept while the cage stands); with one attempt the cage stands.
    xnew, acc = orc.o_round(2, [1.0, 1.0], pos, r, ids, ids, 0.05, 1, 99, 0, 0)
    assert acc[0] == 255
    assert np.array_equal(xnew[0], pos[0])
    xnew, acc = orc.o_round(2, [1.0, 1.0], pos, r, ids, ids, 0.05, 16, 99, 0, 0)
    assert acc[0] != 0  # phase 0 always rejects inside the cage


def test_single_particle_moves_c_m():
    pos = orc.arr([[0.5, 0.5]])
    xnew, acc = orc.o_round(2, [1.0, 1.0], pos, orc.arr([0.1]), [0], [0], 0.05, 4, 17, 0, 0)
    assert acc[0] == 0
    assert np.linalg.norm(xnew[0] - pos[0]) == pytest.approx(0.05, rel=1e-12)


def test_zero_step_is_identity():
    L, pos, r, ids = _state(2, 100, 0.2, 5)
    xnew, acc = orc.o_round(2, L, pos, r, ids, ids, 0.0, 4, 1, 0, 0)
    assert np.array_equal(xnew, pos)


def test_round_depends_on_key_not_on_storage_order():
    # the parallel round is a function of (state, slot), not of the array order
    L, pos, r, ids = _state(3, 500, 0.3, 8)
    r = r * 1.03
    c_m = 0.1 * r[0]
    a_x, a_acc = orc.o_round(3, L, pos, r, ids, ids, c_m, 6, 77, 1, 3)
    perm = np.random.default_rng(0).permutation(len(r))
    b_x, b_acc = orc.o_round(3, L, pos[perm], r[perm], ids[perm], ids[perm], c_m, 6, 77, 1, 3)
    assert np.array_equal(b_x, a_x[perm]) and np.array_equal(b_acc, a_acc[perm])
