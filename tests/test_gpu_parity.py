"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and the
reference, on the same seeded inputs.  Bit-exact for keys, order, offsets, counts,
accept decisions and positions (the kernels are compiled with --fmad=false and use
only correctly rounded operations); max penetration bit-exact too."""
import ctypes as C

import numpy as np
import pytest

import orc
import paper_2605_18254_b200 as srm
from paper_2605_18254_b200 import _native

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["", "lane", "trials", "team", "wave", "resolve"])
def sweep_kernel(request, monkeypatch):
    """Every test once per sweep kernel (SRM_B200_SWEEP: "" = chosen by the grid, lane =
    k_sweep_warpq, trials = k_sweep_trials, team = k_sweep_team, wave = the one-launch wavefront
    k_sweep_wave where the grid allows it): each is exact on any grid."""
    if request.param:
        monkeypatch.setenv("SRM_B200_SWEEP", request.param)
    else:
        monkeypatch.delenv("SRM_B200_SWEEP", raising=False)
    return request.param


def _ctx(L, pos, r, ids=None):
    ctx = srm.Context(L, max(len(r), 1))
    ctx.upload(pos, r, ids)
    return ctx


def _rsa_state(dim, n, f, seed, L=None, poly=False):
    L = L or [1.0] * dim
    unit = np.pi if dim == 2 else 4.0 / 3.0 * np.pi
    if poly:
        rng = np.random.default_rng(seed)
        rel = np.clip(rng.lognormal(-0.5 * np.log(1.04), np.sqrt(np.log(1.04)), n), 0.5, 2.0)
        scale = (f * np.prod(L) / (unit * np.sum(rel ** dim))) ** (1.0 / dim)
        r = rel * scale
    else:
        r = np.full(n, (f * np.prod(L) / (n * unit)) ** (1.0 / dim))
    pos, ids = srm.rsa_place(r, L, 10000, seed)
    return L, pos, r, ids


# ---- primitives -------------------------------------------------------------------
def test_philox_device_vs_curand_and_oracle():
    rng = np.random.default_rng(1)
    n = 4096
    ctr = rng.integers(0, 2**32, size=(n, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2**32, size=(n, 2), dtype=np.uint64).astype(np.uint32)
    ctr[0] = 0; key[0] = 0
    mine = np.zeros((n, 4), np.uint32)
    cur = np.zeros((n, 4), np.uint32)
    assert _native.lib().srm_b200_selftest_philox(n, orc.P(ctr), orc.P(key), orc.P(mine), orc.P(cur)) == 0
    assert np.array_equal(mine, cur)
    for i in range(0, n, 97):
        assert np.array_equal(mine[i], orc.o_philox(ctr[i], key[i]))
    assert tuple(mine[0]) == (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)


@pytest.mark.parametrize("dim", [2, 3])
def test_unit_vectors_bitwise(dim):
    n = 3000
    slot = np.arange(n, dtype=np.uint32) * 7919
    att = (np.arange(n, dtype=np.uint32) % 11)
    out = np.zeros((n, dim))
    seed = 0xDEADBEEF12345678
    assert _native.lib().srm_b200_selftest_unit_vectors(dim, seed, n, orc.P(slot), orc.P(att), 0, 5, 42,
                                                         orc.P(out)) == 0
    exp = np.array([orc.o_unit_vector(dim, seed, int(s), int(a), 0, 5, 42) for s, a in zip(slot, att)])
    assert np.array_equal(out, exp)


# ---- grid rebuild -------------------------------------------------------------------------
@pytest.mark.parametrize("dim,n,cs,L", [
    (2, 5000, 0.013, [1.0, 1.0]), (3, 20000, 0.02, [1.0, 1.0, 1.0]), (3, 3000, 0.4, [1.0, 1.0, 1.0]),
    (2, 777, 0.05, [2.0, 1.0]), (3, 10000, 0.05, [1.0, 1.3, 0.7]), (2, 1, 0.1, [1.0, 1.0]),
])
def test_grid_build_bit_exact(dim, n, cs, L):
    pos, r = orc.random_particles(n, dim, 0.001, 0.002, L, 21)
    if n > 3:
        pos[0, 0] = -1e-9
        pos[1, 0] = np.nextafter(L[0], 0)
        pos[2, :] = 0.0
    with _ctx(L, pos, r) as ctx:
        keys, order, cell_start = ctx.grid_build(cs)
    k_o, dims, _ = orc.o_keys(dim, L, cs, pos)
    assert np.array_equal(keys, k_o)
    k_r, _ = orc.r_keys(dim, L, cs, pos)
    assert np.array_equal(keys.astype(np.uint64), k_r)
    o_order, o_cs = orc.o_sort(k_o, np.arange(n, dtype=np.int32), int(np.prod(dims)))
    assert np.array_equal(order, o_order)
    assert np.array_equal(cell_start, o_cs)
    # == reorder_by_locality of the reference
    _, _, _, remap = orc.r_reorder(dim, L, cs, pos, r, np.arange(n, dtype=np.int32))
    assert np.array_equal(remap[order], np.arange(n))


@pytest.mark.parametrize("dim,cs,L", [(3, 0.0123, [1.0, 1.0, 1.0]), (2, 0.0371, [2.0, 1.0]), (3, 0.05, [1.0, 1.3, 0.7])])
def test_keys_on_cell_boundaries_bit_exact(dim, cs, L):
    """cell_of takes floor(p / edge) from a reciprocal product unless that product is within
    1e-9 of an integer; coordinates on, and a few ulps around, every cell boundary must give
    the reference's keys (floor of the correctly rounded quotient, cell_grid.hpp:62-79)."""
    dims, edge = orc.o_grid(dim, L, cs)
    rows = []
    rng = np.random.default_rng(5)
    for a in range(dim):
        b = np.arange(dims[a] + 1) * edge[a]           # the boundaries as the grid computes them
        b = np.concatenate([b, np.arange(dims[a] + 1) * (L[a] / dims[a]), np.linspace(0.0, L[a], dims[a] + 1)])
        for k in range(-3, 4):
            x = b.copy()
            for _ in range(abs(k)):
                x = np.nextafter(x, np.inf if k > 0 else -np.inf)
            x = x[(x >= 0.0) & (x < L[a])]
            p = rng.uniform(0.0, 1.0, (len(x), dim)) * np.array(L)
            p[:, a] = x
            rows.append(p)
    pos = np.concatenate(rows)
    r = np.full(len(pos), 0.001)
    with _ctx(L, pos, r) as ctx:
        keys, _, _ = ctx.grid_build(cs)
    k_o, _, _ = orc.o_keys(dim, L, cs, pos)
    assert np.array_equal(keys, k_o)
    k_r, _ = orc.r_keys(dim, L, cs, pos)
    assert np.array_equal(keys.astype(np.uint64), k_r)


def test_reorder_by_locality_matches_reference():
    L = [1.0, 1.0, 1.0]
    pos, r = orc.random_particles(4000, 3, 0.001, 0.002, L, 5)
    snap = srm.Snapshot(L, pos, r)
    remap = srm.reorder_by_locality(snap, 0.07)
    pos_r, r_r, ids_r, remap_r = orc.r_reorder(3, L, 0.07, pos, r, np.arange(4000, dtype=np.int32))
    assert np.array_equal(remap, remap_r)
    assert np.array_equal(snap.pos, pos_r) and np.array_equal(snap.radius, r_r)
    assert np.array_equal(snap.id, ids_r)


# ---- overlap reduction --------------------------------------------------------------------
@pytest.mark.parametrize("dim,n,rmin,rmax,seed", [(2, 200, 0.005, 0.02, 11), (3, 3000, 0.005, 0.02, 12),
                                                  (2, 20000, 0.001, 0.004, 13), (3, 500, 0.0, 0.0, 14)])
def test_overlap_stats_bit_exact(dim, n, rmin, rmax, seed):
    L = [1.0] * dim
    pos, r = orc.random_particles(n, dim, rmin, rmax, L, seed)
    if rmax == 0.0:  # coincident points (contact at distance 0), duplicate ids ignored
        r[:] = 0.001
        pos[1] = pos[0]
    cs = 2.5 * r.max()
    with _ctx(L, pos, r) as ctx:
        st = ctx.overlap_stats(cs)
    o = orc.o_stats(dim, L, pos, r)
    assert st.overlap_pairs == o.overlap_pairs
    assert st.max_penetration == o.max_penetration
    keys, dims, _ = orc.o_keys(dim, L, cs, pos)
    assert st.candidate_pairs == orc.o_candidates(dim, dims, keys)
    anyc, _ = orc.r_collisions(dim, L, cs, pos, r)
    assert (st.overlap_pairs > 0) == anyc


# ---- one round (coloured Gauss-Seidel sweep) --------------------------------------------------
@pytest.mark.parametrize("dim,n,f,swell,cm_rel,n_l,seed", [
    (2, 2000, 0.45, 1.03, 0.1, 10, 1),
    (3, 3000, 0.3, 1.02, 0.1, 10, 2),
    (3, 2000, 0.25, 1.06, 0.5, 8, 3),
    (2, 1500, 0.6, 1.0, 0.05, 4, 4),
    (3, 5000, 0.3, 1.0, 0.05, 1, 5),
])
def test_round_bit_exact_vs_oracle(dim, n, f, swell, cm_rel, n_l, seed):
    L, pos, r, ids = _rsa_state(dim, n, min(f, 0.45 if dim == 2 else 0.25), seed)
    r = r * (f / min(f, 0.45 if dim == 2 else 0.25)) ** (1 / dim) * swell
    c_m = cm_rel * r.max()
    cs = 2.5 * r.max() / swell + c_m
    key, round_id, it = 0x0123456789ABCDEF + seed, 3, 17
    with _ctx(L, pos, r, ids) as ctx:
        st, acc = ctx.round(cs, c_m, n_l, key, round_id, it, with_candidates=True)
        pos_d, r_d, id_d = ctx.download()
    xnew, acc_o = orc.o_round(dim, L, pos, r, ids, ids, cs, c_m, n_l, key, round_id, it)
    assert np.array_equal(acc, acc_o)
    assert np.array_equal(pos_d, xnew)
    assert np.array_equal(r_d, r) and np.array_equal(id_d, ids)
    o = orc.o_stats(dim, L, xnew, r)
    assert st.overlap_pairs == o.overlap_pairs
    assert st.max_penetration == o.max_penetration
    assert st.movers == int(np.sum(acc_o != 255))
    keys, dims, _ = orc.o_keys(dim, L, cs, pos)
    assert st.candidate_pairs == orc.o_candidates(dim, dims, keys)


@pytest.mark.parametrize("dim,n,L,cm_rel,swell", [
    (3, 400, [1.0, 1.0, 1.0], 0.1, 1.02),      # dims 3-4: whole axes, every coordinate its own colour
    (3, 3000, [2.0, 1.0, 0.5], 0.1, 1.03),     # rectangular, odd dims: tail colours
    (3, 4000, [1.0, 1.0, 1.0], 0.45, 1.05),    # wide moves: colouring modulus 3, near half width 2
    (2, 6000, [1.0, 3.0], 0.2, 1.02),
    (2, 300, [1.0, 1.0], 0.3, 1.0),
])
def test_round_colourings_bit_exact(dim, n, L, cm_rel, swell):
    unit = np.pi if dim == 2 else 4.0 / 3.0 * np.pi
    f = 0.35 if dim == 2 else 0.2
    r = (f * np.prod(L) / (n * unit)) ** (1.0 / dim)
    pos, ids = srm.rsa_place(np.full(n, r), L, 10000, 31)
    rr = np.full(n, r * swell)
    c_m = cm_rel * r
    cs = 2.5 * r + c_m
    with _ctx(L, pos, rr, ids) as ctx:
        st, acc = ctx.round(cs, c_m, 6, 4242, 1, 2, with_candidates=True)
        pos_d, _, _ = ctx.download()
        info = ctx.last_round_info()
    xnew, acc_o = orc.o_round(dim, L, pos, rr, ids, ids, cs, c_m, 6, 4242, 1, 2)
    assert np.array_equal(acc, acc_o) and np.array_equal(pos_d, xnew)
    o = orc.o_stats(dim, L, xnew, rr)
    assert st.overlap_pairs == o.overlap_pairs and st.max_penetration == o.max_penetration
    assert info["nonmovers"] == int(np.sum(acc_o == 255))
    m, ncol = orc.o_colouring(dim, L, cs, rr.max(), c_m)
    assert info["colour_classes"] == int(np.prod(ncol))


def test_clustered_start_bit_exact():
    # dense Gaussian clusters (cfg3-like start): many particles per cell, long in-cell
    # sequential chains and near lists beyond the per-particle buffer
    rng = np.random.default_rng(8)
    n, L = 6000, [1.0, 1.0, 1.0]
    centres = rng.uniform(0, 1, (6, 3))
    pos = np.mod(centres[np.arange(n) % 6] + rng.normal(0, 0.04, (n, 3)), 1.0)
    r = np.full(n, 0.0035)
    c_m = 0.1 * r[0]
    cs = 2.5 * r[0] + c_m
    with _ctx(L, pos, r) as ctx:
        st, acc = ctx.round(cs, c_m, 5, 7, 0, 0)
        pos_d, _, _ = ctx.download()
    xnew, acc_o = orc.o_round(3, L, pos, r, np.arange(n, dtype=np.int32), np.arange(n, dtype=np.int32),
                              cs, c_m, 5, 7, 0, 0)
    assert np.array_equal(acc, acc_o) and np.array_equal(pos_d, xnew)
    assert st.overlap_pairs == orc.o_stats(3, L, xnew, r).overlap_pairs


def test_round_polydisperse_bit_exact():
    L, pos, r, ids = _rsa_state(3, 4000, 0.22, 9, L=[1.0, 1.0, 1.0], poly=True)
    r = r * 1.04
    c_m = 0.1 * np.mean(r)
    cs = 2.5 * r.max() / 1.04 + c_m
    with _ctx(L, pos, r, ids) as ctx:
        st, acc = ctx.round(cs, c_m, 10, 99, 0, 1)
        pos_d, _, _ = ctx.download()
    xnew, acc_o = orc.o_round(3, L, pos, r, ids, ids, cs, c_m, 10, 99, 0, 1)
    assert np.array_equal(acc, acc_o) and np.array_equal(pos_d, xnew)
    assert st.overlap_pairs == orc.o_stats(3, L, xnew, r).overlap_pairs


@pytest.mark.parametrize("swell,n_l,seed", [(1.03, 10, 21), (1.12, 4, 22)])
def test_round_crowded_spheres_team_sweep(swell, n_l, seed):
    """Bidisperse spheres (1 in 20 four times larger): the cell edge follows the large
    radius, so a cell holds ~16 particles -- the crowded near kind (4x4x4 bricks, lists in
    the overflow pool) and the team sweep (k_sweep_team: a team of lanes per cell splits
    each trial's candidates).  Two rounds, bit for bit against the oracle."""
    n, nl, L = 12000, 600, [1.0, 1.0, 1.0]
    rel = np.ones(n)
    rel[:nl] = 4.0  # placed first
    rs = (0.2 / (4.0 / 3.0 * np.pi * np.sum(rel ** 3))) ** (1.0 / 3.0)
    r0 = rel * rs
    pos, ids = srm.rsa_place(r0, L, 100000, seed)
    r = r0 * swell
    c_m = 0.1 * np.mean(r)
    cs = 2.5 * r.max() / swell + c_m
    key = 0x5EED + seed
    with srm.Context(L, n) as ctx:
        ctx.upload(pos, r, ids)
        for rid in range(2):
            st, acc = ctx.round(cs, c_m, n_l, key, rid, 3)
        info = ctx.last_round_info()
        p_d, _, _ = ctx.download()
    assert n > 1.8 * info["cells"] and info["cells"] >= 6 ** 3  # the crowded kind
    x = pos
    for rid in range(2):
        x, ao = orc.o_round(3, L, x, r, ids, ids, cs, c_m, n_l, key, rid, 3)
    assert np.array_equal(acc, ao)
    assert np.array_equal(p_d, x)
    o = orc.o_stats(3, L, x, r)
    assert st.overlap_pairs == o.overlap_pairs and st.max_penetration == o.max_penetration


def test_rounds_are_deterministic_and_chain():
    L, pos, r, ids = _rsa_state(3, 6000, 0.3, 7)
    r = r * 1.02
    c_m = 0.1 * r[0]
    cs = 2.5 * r[0] / 1.02 + c_m
    outs = []
    for _ in range(2):
        with _ctx(L, pos, r, ids) as ctx:
            ctx.rounds(cs, c_m, 10, 5, 0, 1, 3)
            outs.append(ctx.download()[0])
    assert np.array_equal(outs[0], outs[1])
    x = pos
    for k in range(3):
        x, _ = orc.o_round(3, L, x, r, ids, ids, cs, c_m, 10, 5, k, 1)
    assert np.array_equal(outs[0], x)


def test_caged_particle_reverts():
    # test_engine.cpp:65-86: a particle that rejects keeps its exact bits
    pos = orc.arr([[0.5, 0.5]] + [[0.5 + 0.2000000001 * np.cos(k * np.pi / 3),
                                     0.5 + 0.2000000001 * np.sin(k * np.pi / 3)] for k in range(6)])
    r = np.full(7, 0.1)
    with _ctx([1.0, 1.0], pos, r) as ctx:
        _, acc = ctx.round(0.25, 0.05, 1, 99, 0, 0)
        p, _, _ = ctx.download()
    xnew, acc_o = orc.o_round(2, [1.0, 1.0], pos, r, np.arange(7, dtype=np.int32), np.arange(7, dtype=np.int32),
                              0.25, 0.05, 1, 99, 0, 0)
    assert np.array_equal(acc, acc_o) and np.array_equal(p, xnew)
    for i in range(7):
        if acc[i] == 255:
            assert np.array_equal(p[i], pos[i])


def test_single_particle_moves_c_m():
    with _ctx([1.0, 1.0], orc.arr([[0.5, 0.5]]), orc.arr([0.1])) as ctx:
        _, acc = ctx.round(0.25, 0.05, 4, 17, 0, 0)
        p, _, _ = ctx.download()
    assert acc[0] == 0
    assert np.linalg.norm(p[0] - [0.5, 0.5]) == pytest.approx(0.05, rel=1e-12)


def test_records_roundtrip():
    # std::vector<srm::Particle<3>> layout: int id @0, double pos[3] @8, radius @32, stride 40
    dt = np.dtype({"names": ["id", "pos", "radius"], "formats": ["<i4", ("<f8", 3), "<f8"],
                   "offsets": [0, 8, 32], "itemsize": 40})
    L = [1.0, 1.0, 1.0]
    pos, r = orc.random_particles(1000, 3, 0.001, 0.002, L, 3)
    rec = np.zeros(1000, dt)
    rec["id"] = np.arange(1000)[::-1]
    rec["pos"] = pos
    rec["radius"] = r
    ctx = srm.Context(L, 1000)
    ctx.upload_records(rec, 0, 8, 32)
    ctx.grid_build(0.05)  # permutes the device copy
    out = np.zeros(1000, dt)
    ctx.download_records(out, 0, 8, 32)
    ctx.close()
    assert np.array_equal(out["pos"], pos) and np.array_equal(out["radius"], r)
    assert np.array_equal(out["id"], rec["id"])


# ---- the large-grid kernels: shared-memory near-list bricks, the overflow pool ------------
@pytest.mark.parametrize("n,f,swell,cm_rel,poly,seed", [
    (40000, 0.25, 1.03, 0.05, False, 11),   # k_near_tiles (>= 18 x 10 x 6 cells, one-cell stencil)
    (30000, 0.15, 1.05, 0.6, True, 12),     # polydisperse, long reach: crowded rows -> overflow pool
    (60000, 0.3, 1.0, 0.02, False, 13),     # dense, small steps
])
def test_round_bit_exact_large_grids(n, f, swell, cm_rel, poly, seed):
    L, pos, r, ids = _rsa_state(3, n, f, seed, poly=poly)
    r = r * swell
    c_m = cm_rel * r.max()
    cs = 2.5 * r.max() / swell + c_m
    with srm.Context(L, n) as ctx:
        ctx.upload(pos, r, ids)
        st, acc = ctx.round(cs, c_m, 10, 0xABC + seed, 3, 7)
        p_d, r_d, id_d = ctx.download()
        info = ctx.last_round_info()
    xo, ao = orc.o_round(3, L, pos, r, ids, ids, cs, c_m, 10, 0xABC + seed, 3, 7)
    assert np.array_equal(acc, ao)
    assert np.array_equal(p_d, xo)
    o = orc.o_stats(3, L, xo, r)
    assert st.overlap_pairs == o.overlap_pairs and st.max_penetration == o.max_penetration
    if not poly:
        assert min(info["cells"], 10 ** 9) >= 18 * 10 * 6  # large enough for the bricks
