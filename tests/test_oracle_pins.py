"""Pin the CPU oracle (oracle/srm_oracle.c) to the reference.

Two kinds of pins, per SURVEY.md §8c:
  * the reference's own known-answer cases (test_geometry.cpp, test_cell_grid.cpp,
    test_engine.cpp), re-expressed against the oracle AND the compiled reference;
  * agreement with the reference's functions (oracle/_ref/libsrm_ref.so, built from
    /root/reference sources) on seeded states: cell keys (CellGrid::cell_of), sorted
    order (reorder_by_locality), collision booleans (check_particle_collision /
    shape_any_collision);
  * Philox4x32-10 against the Random123 known-answer vectors.
"""
import numpy as np
import pytest

import orc


# ---- geometry: test_geometry.cpp:31-62 ---------------------------------------------
@pytest.mark.parametrize("impl", ["oracle", "ref"])
def test_wrap_cases(impl):
    def wrap(p, L=(1.0, 1.0)):
        p = orc.arr(p).copy()
        (orc.orc().orc_wrap if impl == "oracle" else orc.ref().ref_wrap)(2, orc.P(orc.arr(L)), orc.P(p))
        return p

    assert wrap([-0.05, 0.5])[0] == pytest.approx(0.95)
    assert wrap([0.3, 0.5])[0] == 0.3
    assert wrap([1.0, 0.5])[0] == 0.0
    w = wrap([-1e-300, 0.0])  # rounds up to exactly L, must land at 0 (test_geometry.cpp:38-46)
    assert w[0] == 0.0 and not np.signbit(w[0]) or w[0] == 0.0


@pytest.mark.parametrize("impl", ["oracle", "ref"])
def test_min_image_cases(impl):
    f = orc.orc().orc_min_image_dist2 if impl == "oracle" else orc.ref().ref_min_image_dist2
    L = orc.arr([10.0, 10.0])

    def d2(a, b):
        return f(2, orc.P(L), orc.P(orc.arr(a)), orc.P(orc.arr(b)))

    assert d2([0.5, 0.0], [9.5, 0.0]) == pytest.approx(1.0)
    assert d2([3.0, 0.0], [1.0, 0.0]) == pytest.approx(4.0)
    assert np.sqrt(d2([0.1, 0.1], [9.9, 9.9])) == pytest.approx(0.2 * np.sqrt(2.0))
    L2 = orc.arr([2.0, 2.0])
    assert f(2, orc.P(L2), orc.P(orc.arr([1.5, 0.0])), orc.P(orc.arr([0.5, 0.0]))) == 1.0  # half box


def test_min_image_bitwise_vs_ref():
    rng = np.random.default_rng(5)
    for dim in (2, 3):
        L = orc.arr(rng.uniform(0.5, 3.0, dim))
        for _ in range(2000):
            a = orc.arr(rng.uniform(0, 1, dim) * L)
            b = orc.arr(rng.uniform(0, 1, dim) * L)
            o = orc.orc().orc_min_image_dist2(dim, orc.P(L), orc.P(a), orc.P(b))
            r = orc.ref().ref_min_image_dist2(dim, orc.P(L), orc.P(a), orc.P(b))
            assert o == r


# ---- grid: test_cell_grid.cpp:13-55 -----------------------------------------------
def test_grid_dims_cases():
    dims, _ = orc.o_grid(2, [1.0, 1.0], 2.5 * 0.01 + 0.005)
    assert list(dims) == [33, 33]
    dims, _ = orc.o_grid(2, [1.0, 1.0], 0.5)
    assert dims[0] == 3  # floor(2) clamped to 3
    dims, _ = orc.o_grid(2, [2.0, 1.0], 0.1)
    assert list(dims) == [20, 10]
    with pytest.raises(ValueError):
        orc.o_grid(2, [1.0, 1.0], 0.0)


def test_grid_safety_bound_ref():
    d = np.zeros(3, np.int32)
    e = np.zeros(3)
    L = orc.arr([1.0, 1.0])
    assert orc.ref().ref_grid_dims(2, orc.P(L), 0.02, 0.01, 0.005, 1, orc.P(d), orc.P(e)) == 1
    assert orc.ref().ref_grid_dims(2, orc.P(L), 0.0, 0.0, 0.0, 0, orc.P(d), orc.P(e)) == 1
    assert orc.ref().ref_grid_dims(2, orc.P(L), 0.025, 0.01, 0.005, 1, orc.P(d), orc.P(e)) == 0


def test_cell_coords_cases():
    dims, edge = orc.o_grid(2, [1.0, 1.0], 0.1)
    assert dims[0] == 10

    def coords(p):
        c = np.zeros(3, np.int32)
        orc.orc().orc_cell_coords(2, orc.P(orc.arr(dims, np.int32)), orc.P(orc.arr(edge)), orc.P(orc.arr(p)), orc.P(c))
        return list(c[:2])

    assert coords([0.0, 0.0])[0] == 0
    assert coords([-1e-9, 0.0])[0] == 9
    assert coords([0.999, 0.0])[0] == 9
    assert coords([0.35, 0.75]) == [3, 7]
    # the reference agrees on the same points
    pts = orc.arr([[0.0, 0.0], [-1e-9, 0.0], [0.999, 0.0], [0.35, 0.75]])
    _, rc = orc.r_keys(2, [1.0, 1.0], 0.1, pts)
    assert [list(v) for v in rc] == [[0, 0], [9, 0], [9, 0], [3, 7]]


def test_flat_index_row_major():
    dims, edge = orc.o_grid(3, [2.0, 1.0, 1.0], 0.1)
    assert list(dims) == [20, 10, 10]

    def key(c):
        p = (np.asarray(c) + 0.5) * edge
        return orc.orc().orc_cell_of(3, orc.P(orc.arr(dims, np.int32)), orc.P(orc.arr(edge)), orc.P(orc.arr(p)))

    assert key([0, 0, 0]) == 0
    assert key([1, 0, 0]) == 1
    assert key([0, 1, 0]) == 20
    assert key([0, 0, 1]) == 200


@pytest.mark.parametrize("dim,n,cs,seed", [(2, 3000, 0.013, 1), (3, 3000, 0.07, 2), (2, 500, 0.4, 3),
                                           (3, 2000, 0.011, 4)])
def test_keys_match_reference(dim, n, cs, seed):
    L = [1.0, 0.8, 1.3][:dim]
    pos, r = orc.random_particles(n, dim, 0.001, 0.002, L, seed)
    # include the boundary-rounding cases the reference cares about
    pos[0, 0] = -1e-9
    pos[1, 0] = L[0] - 1e-17
    pos[2, :] = 0.0
    k_o, dims, _ = orc.o_keys(dim, L, cs, pos)
    k_r, _ = orc.r_keys(dim, L, cs, pos)
    assert np.array_equal(k_o.astype(np.uint64), k_r)


@pytest.mark.parametrize("dim,n,cs,seed", [(2, 2000, 0.02, 7), (3, 2000, 0.08, 8), (2, 300, 0.4, 9)])
def test_sort_order_matches_reorder_by_locality(dim, n, cs, seed):
    L = [1.0] * dim
    pos, r = orc.random_particles(n, dim, 0.001, 0.002, L, seed)
    ids = np.arange(n, dtype=np.int32)
    keys, dims, _ = orc.o_keys(dim, L, cs, pos)
    ncells = int(np.prod(dims))
    order, cell_start = orc.o_sort(keys, ids, ncells)
    pos_r, r_r, ids_r, remap = orc.r_reorder(dim, L, cs, pos, r, ids)
    # reference: remap[old] = new; sorted position q holds old index order[q]
    assert np.array_equal(remap[order], np.arange(n))
    assert np.array_equal(pos_r, pos[order])
    assert np.array_equal(ids_r, np.arange(n))
    assert cell_start[-1] == n
    assert np.all(np.diff(cell_start) >= 0)
    assert np.array_equal(np.bincount(keys, minlength=ncells), np.diff(cell_start))


def test_reorder_identity_and_reverse():
    # test_engine.cpp:114-142: one particle per cell in row-major order is sorted
    L = [1.0, 1.0]
    dims, _ = orc.o_grid(2, L, 0.25)
    d = dims[0]
    pos = orc.arr([[(x + 0.5) / d, (y + 0.5) / d] for y in range(d) for x in range(d)])
    keys, _, _ = orc.o_keys(2, L, 0.25, pos)
    order, _ = orc.o_sort(keys, np.arange(len(pos), dtype=np.int32), int(np.prod(dims)))
    assert np.array_equal(order, np.arange(len(pos)))
    rev = pos[::-1].copy()
    keys, _, _ = orc.o_keys(2, L, 0.25, rev)
    order, _ = orc.o_sort(keys, np.arange(len(pos), dtype=np.int32), int(np.prod(dims)))
    assert np.array_equal(rev[order], pos)


# ---- collisions: test_cell_grid.cpp:97-162 ---------------------------------------------
def test_pair_collision_cases():
    L = [1.0, 1.0]
    r = orc.arr([0.1, 0.1])
    assert orc.o_stats(2, L, [[0.40, 0.5], [0.55, 0.5]], r).overlap_pairs == 1
    assert orc.o_stats(2, L, [[0.40, 0.5], [0.65, 0.5]], r).overlap_pairs == 0
    assert orc.o_stats(2, L, [[0.05, 0.5], [0.95, 0.5]], r).overlap_pairs == 1  # across the seam
    # exact contact counts as overlap
    st = orc.o_stats(2, L, [[0.25, 0.5], [0.5, 0.5]], orc.arr([0.125, 0.125]))
    assert st.overlap_pairs == 1 and st.max_penetration == 0.0


@pytest.mark.parametrize("dim,seed", [(2, 11), (3, 12)])
def test_collisions_match_reference(dim, seed):
    # test_cell_grid.cpp:116-132: 200 particles, r in [0.005, 0.02], Rng(11)
    L = [1.0] * dim
    n = 200 if dim == 2 else 400
    rmax = 0.02 if dim == 2 else 0.04
    pos, r = orc.random_particles(n, dim, 0.005, rmax, L, seed)
    anyc, per = orc.r_collisions(dim, L, 2.5 * rmax, pos, r)
    st = orc.o_stats(dim, L, pos, r)
    assert (st.overlap_pairs > 0) == anyc
    # per-particle brute force with the oracle predicate == reference cell-list query
    for i in range(n):
        hit = False
        for j in range(n):
            if j == i:
                continue
            rr = r[i] + r[j]
            d2 = orc.orc().orc_min_image_dist2(dim, orc.P(orc.arr(L)), orc.P(pos[i].copy()), orc.P(pos[j].copy()))
            if d2 <= rr * rr:
                hit = True
                break
        assert hit == bool(per[i])


def test_candidate_pairs_definition():
    # brute-force count of ordered (i, j != i) pairs whose cells are 3^d neighbours
    for dim, cs in ((2, 0.1), (3, 0.2), (2, 0.45)):
        L = [1.0] * dim
        pos, r = orc.random_particles(300, dim, 0.01, 0.01, L, 5)
        keys, dims, _ = orc.o_keys(dim, L, cs, pos)
        coords = np.stack(np.unravel_index(keys.astype(np.int64), tuple(dims[::-1]))[::-1], axis=1)
        cnt = 0
        for i in range(len(pos)):
            dd = np.abs(coords - coords[i])
            dd = np.minimum(dd, dims[None, :] - dd)
            cnt += int(np.sum(np.all(dd <= 1, axis=1))) - 1
        assert orc.o_candidates(dim, dims, keys) == cnt


# ---- RNG ------------------------------------------------------------------------------
def test_philox_random123_kat():
    # Random123 kat_vectors, philox4x32 10 rounds
    kat = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
           ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
           ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
            (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for c, k, o in kat:
        assert tuple(int(v) for v in orc.o_philox(c, k)) == o


def test_unit_vectors_are_unit_and_isotropic():
    for dim in (2, 3):
        us = np.array([orc.o_unit_vector(dim, 123456789, s, a, 0, 3, 7) for s in range(2000) for a in range(2)])
        norms = np.linalg.norm(us, axis=1)
        assert np.max(np.abs(norms - 1.0)) < 4e-16
        assert np.all(np.abs(us.mean(axis=0)) < 0.05)
        # mean |u . e_last| = 1/2 in 3D (uniform on S^2), 2/pi in 2D
        m = np.mean(np.abs(us[:, -1]))
        assert m == pytest.approx(0.5 if dim == 3 else 2 / np.pi, abs=0.02)


def test_mt19937_64_pinned():
    # std::mt19937_64 is pinned by the C++ standard: the 10000th draw of the default
    # seed (5489) is 9981545732273789042 ([rand.predef]).
    out = np.zeros(10000, np.uint64)
    orc.ref().ref_rng_raw(5489, 10000, orc.P(out))
    assert int(out[-1]) == 9981545732273789042
