"""ctypes wrappers for the CPU checkers (test infrastructure only).

  oracle/liboracle.so          plain-C restatement (oracle/srm_oracle.c)
  oracle/_ref/libsrm_ref.so    the reference's own headers compiled where they lie
                               (oracle/ref_harness.cpp + oracle/Makefile)
Both are built by ``make oracle`` / __graft_entry__.build() in the build container and
travel to the GPU box as prebuilt files; nothing here reads /root/reference.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libsrm_ref.so")

dp = C.POINTER(C.c_double)
vp = C.c_void_p


def P(a):
    # data_as keeps a reference to the array, so temporaries stay alive for the call
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class RoundStats(C.Structure):
    _fields_ = [("overlap_pairs", C.c_int64), ("max_penetration", C.c_double),
                ("candidate_pairs", C.c_int64), ("movers", C.c_int64)]


_orc = None
_ref = None


def orc():
    global _orc
    if _orc is None:
        L = C.CDLL(ORACLE_SO)
        L.orc_wrap.argtypes = [C.c_int, vp, vp]
        L.orc_min_image_dist2.restype = C.c_double
        L.orc_min_image_dist2.argtypes = [C.c_int, vp, vp, vp]
        L.orc_grid_dims.restype = C.c_int
        L.orc_grid_dims.argtypes = [C.c_int, vp, C.c_double, vp, vp]
        L.orc_cell_coords.argtypes = [C.c_int, vp, vp, vp, vp]
        L.orc_cell_of.restype = C.c_uint64
        L.orc_cell_of.argtypes = [C.c_int, vp, vp, vp]
        L.orc_keys.argtypes = [C.c_int, vp, vp, C.c_int64, vp, vp]
        L.orc_sort_by_cell.argtypes = [C.c_int64, vp, vp, C.c_int64, vp, vp]
        L.orc_philox4x32_10.argtypes = [vp, vp, vp]
        L.orc_unit_vector.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                      C.c_uint32, C.c_uint32, vp]
        L.orc_propose.argtypes = [C.c_int, vp, vp, C.c_double, C.c_uint64, C.c_uint32, C.c_uint32,
                                  C.c_uint32, C.c_uint32, vp]
        L.orc_sweep_round.argtypes = [C.c_int, vp, C.c_int64, vp, vp, vp, vp, C.c_double, C.c_double, C.c_int,
                                      C.c_uint64, C.c_uint32, C.c_uint32, vp, vp, C.c_int]
        L.orc_colouring.argtypes = [C.c_int, vp, vp, C.c_double, C.c_double, vp, vp]
        L.orc_overlap_stats.argtypes = [C.c_int, vp, C.c_int64, vp, vp, vp, C.POINTER(RoundStats)]
        L.orc_candidate_pairs.restype = C.c_int64
        L.orc_candidate_pairs.argtypes = [C.c_int, vp, C.c_int64, vp]
        L.orc_max_radius.restype = C.c_double
        L.orc_max_radius.argtypes = [C.c_int64, vp]
        L.orc_volume_fraction_seq.restype = C.c_double
        L.orc_volume_fraction_seq.argtypes = [C.c_int, vp, C.c_int64, vp]
        d = C.c_double
        L.orc_pl_overlap.restype = C.c_int
        L.orc_pl_overlap.argtypes = [vp, vp, vp, d, d, vp, vp, d, d]
        L.orc_pl_disks_within.restype = d
        L.orc_pl_disks_within.argtypes = [vp, vp, d, vp, vp, d, d]
        L.orc_pl_measure.restype = d
        L.orc_pl_measure.argtypes = [d, d]
        L.orc_pl_propose.argtypes = [vp, vp, vp, d, d, d, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                     vp, vp]
        L.orc_pl_sweep_round.argtypes = [vp, C.c_int64, vp, vp, vp, vp, vp, vp, d, d, d, d, C.c_int, C.c_uint64,
                                         C.c_uint32, C.c_uint32, vp, vp, vp]
        L.orc_pl_overlap_pairs.restype = C.c_int64
        L.orc_pl_overlap_pairs.argtypes = [vp, C.c_int64, vp, vp, vp, vp, vp]
        _orc = L
    return _orc


def ref():
    global _ref
    if _ref is None:
        L = C.CDLL(REF_SO)
        L.ref_mix_seed.restype = C.c_uint64
        L.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_rng_uniforms.argtypes = [C.c_uint64, C.c_int64, vp]
        L.ref_rng_raw.argtypes = [C.c_uint64, C.c_int64, vp]
        L.ref_wrap.argtypes = [C.c_int, vp, vp]
        L.ref_min_image_dist2.restype = C.c_double
        L.ref_min_image_dist2.argtypes = [C.c_int, vp, vp, vp]
        L.ref_grid_dims.restype = C.c_int
        L.ref_grid_dims.argtypes = [C.c_int, vp, C.c_double, C.c_double, C.c_double, C.c_int, vp, vp]
        L.ref_cell_keys.argtypes = [C.c_int, vp, C.c_double, C.c_int64, vp, vp, vp]
        L.ref_reorder.argtypes = [C.c_int, vp, C.c_double, C.c_int64, vp, vp, vp, vp]
        L.ref_collisions.restype = C.c_int
        L.ref_collisions.argtypes = [C.c_int, vp, C.c_double, C.c_int64, vp, vp, vp, vp]
        L.ref_rsa_place.restype = C.c_int
        L.ref_rsa_place.argtypes = [C.c_int, vp, C.c_int64, vp, C.c_int64, C.c_uint64, vp, vp, vp]
        L.ref_generate.restype = C.c_int
        L.ref_generate.argtypes = [C.c_int, vp, C.c_int64, vp, vp, vp, C.c_double, C.c_double, C.c_int,
                                   C.c_int, C.c_double, C.c_int64, C.c_uint64, C.c_int, vp, vp, vp]
        L.ref_migrate.argtypes = [C.c_int, vp, C.c_int64, vp, vp, vp, C.c_double, C.c_double, C.c_int,
                                  C.c_uint64, vp]
        L.ref_nnd.argtypes = [C.c_int, vp, C.c_int64, vp, vp]
        L.ref_histogram.argtypes = [C.c_int64, vp, C.c_int, C.c_double, C.c_double, vp]
        L.ref_bench_rounds.restype = C.c_double
        L.ref_bench_rounds.argtypes = [C.c_int, vp, C.c_int64, vp, vp, vp, C.c_double, C.c_int, C.c_int,
                                       C.c_uint64, C.c_int, vp]
        d = C.c_double
        L.ref_pl_overlap.restype = C.c_int
        L.ref_pl_overlap.argtypes = [vp, vp, vp, d, d, vp, vp, d, d]
        L.ref_pl_disks_within.restype = C.c_int
        L.ref_pl_disks_within.argtypes = [vp, vp, d, vp, vp, d, d]
        L.ref_pl_disk_distance.restype = d
        L.ref_pl_disk_distance.argtypes = [vp, vp, d, vp, vp, d]
        L.ref_pl_measure.restype = d
        L.ref_pl_measure.argtypes = [d, d]
        L.ref_pl_rotate.argtypes = [vp, vp, d, vp]
        L.ref_rsa_platelets.restype = C.c_int
        L.ref_rsa_platelets.argtypes = [C.c_int64, d, d, vp, C.c_int64, C.c_uint64, vp, vp, vp]
        L.ref_generate_platelets.restype = C.c_int
        L.ref_generate_platelets.argtypes = [vp, C.c_int64, vp, vp, vp, vp, vp, d, d, d, C.c_int, C.c_int, d,
                                             C.c_int64, C.c_uint64, C.c_int, vp, vp]
        L.ref_local_nematic_order.restype = C.c_int
        L.ref_local_nematic_order.argtypes = [vp, C.c_int64, vp, vp, vp, vp, d, vp, vp]
        L.ref_pl_any_collision.restype = C.c_int
        L.ref_pl_any_collision.argtypes = [vp, d, C.c_int64, vp, vp, vp, vp, vp]
        _ref = L
    return _ref


def arr(v, dt=np.float64):
    return np.ascontiguousarray(np.asarray(v, dtype=dt))


# ---- oracle helpers ------------------------------------------------------------------
def o_grid(dim, L, cs):
    dims = np.zeros(3, np.int32)
    edge = np.zeros(3, np.float64)
    rc = orc().orc_grid_dims(dim, P(arr(L)), cs, P(dims), P(edge))
    if rc != 0:
        raise ValueError("cell size must be positive")
    return dims[:dim].copy(), edge[:dim].copy()


def o_keys(dim, L, cs, pos):
    dims, edge = o_grid(dim, L, cs)
    pos = arr(pos)
    keys = np.zeros(len(pos), np.uint32)
    orc().orc_keys(dim, P(dims), P(edge), len(pos), P(pos), P(keys))
    return keys, dims, edge


def o_sort(keys, slot, ncells):
    n = len(keys)
    order = np.zeros(n, np.int32)
    cs = np.zeros(ncells + 1, np.int64)
    orc().orc_sort_by_cell(n, P(arr(keys, np.uint32)), P(arr(slot, np.int32)), ncells, P(order), P(cs))
    return order, cs


def o_round(dim, L, x0, r, ids, slot, cell_size, c_m, n_l, seed, round_id, iteration, brute=False):
    """one round's coloured Gauss-Seidel migrate sweep (oracle/srm_oracle.c)"""
    x0 = arr(x0)
    n = len(r)
    xnew = np.zeros_like(x0)
    acc = np.zeros(n, np.uint8)
    orc().orc_sweep_round(dim, P(arr(L)), n, P(x0), P(arr(r)), P(arr(ids, np.int32)),
                          P(arr(slot, np.int32)), cell_size, c_m, n_l, seed, round_id, iteration,
                          P(xnew), P(acc), int(brute))
    return xnew, acc


def o_colouring(dim, L, cell_size, maxr, c_m):
    dims, edge = o_grid(dim, L, cell_size)
    d3 = np.ones(3, np.int32); d3[:dim] = dims
    e3 = np.ones(3); e3[:dim] = edge
    m = np.zeros(3, np.int32)
    ncol = np.zeros(3, np.int32)
    orc().orc_colouring(dim, P(d3), P(e3), maxr, c_m, P(m), P(ncol))
    return m[:dim].copy(), ncol[:dim].copy()


def o_stats(dim, L, pos, r, ids=None):
    n = len(r)
    ids = np.arange(n, dtype=np.int32) if ids is None else ids
    st = RoundStats()
    orc().orc_overlap_stats(dim, P(arr(L)), n, P(arr(pos)), P(arr(r)), P(arr(ids, np.int32)), C.byref(st))
    return st


def o_candidates(dim, dims, keys):
    return orc().orc_candidate_pairs(dim, P(arr(dims, np.int32)), len(keys), P(arr(keys, np.uint32)))


def o_unit_vector(dim, seed, slot, attempt, stream, round_id, iteration):
    u = np.zeros(3)
    orc().orc_unit_vector(dim, seed, slot, attempt, stream, round_id, iteration, P(u))
    return u[:dim].copy()


def o_philox(ctr, key):
    c = arr(ctr, np.uint32)
    k = arr(key, np.uint32)
    out = np.zeros(4, np.uint32)
    orc().orc_philox4x32_10(P(c), P(k), P(out))
    return out


def o_generate(dim, L, pos, r, ids, c_w, c_m, n_k, n_l, f_target, max_iterations, seed,
               reorder_period=16, iteration_count=0):
    """Oracle restatement of the device srm_generate loop (engine.hpp:176-260 with the
    parallel round).  The volume fraction uses the sequential sum (the device uses a
    fixed tree, equal to ~1e-15), so this is a statistical, not bitwise, oracle for the
    whole loop.  Returns (status, pos, r, ids, iterations, f, stats dict)."""
    pos = arr(pos).copy()
    r = arr(r).copy()
    ids = arr(ids, np.int32).copy()
    slot = np.arange(len(r), dtype=np.int32)
    Lp = P(arr(L))
    f = orc().orc_volume_fraction_seq(dim, Lp, len(r), P(r))
    stop = f_target * (1.0 - 1e-12)
    done = acc_it = rounds = shakes = 0
    status = 0
    while f < stop:
        if done >= max_iterations:
            status = 1
            break
        done += 1
        it = iteration_count + done
        factor = 1.0 + c_w
        if f * factor ** dim > f_target:
            factor = (f_target / f) ** (1.0 / dim)
        max_r = float(r.max())
        cs = 2.5 * max_r + c_m
        q = r * factor
        x = pos
        ok = False
        for k in range(n_k):
            x, _ = o_round(dim, L, x, q, ids, slot, cs, c_m, n_l, seed, k, it & 0xFFFFFFFF)
            rounds += 1
            if o_stats(dim, L, x, q, ids).overlap_pairs == 0:
                ok = True
                break
        if ok:
            pos, r = x, q
            f = orc().orc_volume_fraction_seq(dim, Lp, len(r), P(r))
            acc_it += 1
            # reorder cadence changes slots/ids exactly like reorder_by_locality
            if reorder_period > 0 and acc_it % reorder_period == 0:
                keys, dims, _ = o_keys(dim, L, cs, pos)
                order, _ = o_sort(keys, slot, int(np.prod(dims)))
                pos, r = pos[order], r[order]
                slot = np.arange(len(r), dtype=np.int32)
                ids = slot.copy()
        else:
            for k in range(n_k):
                pos, _ = o_round(dim, L, pos, r, ids, slot, cs, c_m, n_l, seed, n_k + k, it & 0xFFFFFFFF)
                shakes += 1
    return status, pos, r, ids, iteration_count + done, f, dict(accepted=acc_it, rounds=rounds, shakes=shakes)


# ---- reference helpers ---------------------------------------------------------------
def r_keys(dim, L, cs, pos):
    pos = arr(pos)
    keys = np.zeros(len(pos), np.uint64)
    coords = np.zeros((len(pos), dim), np.int32)
    ref().ref_cell_keys(dim, P(arr(L)), cs, len(pos), P(pos), P(keys), P(coords))
    return keys, coords


def r_reorder(dim, L, cs, pos, r, ids):
    pos = arr(pos).copy()
    r = arr(r).copy()
    ids = arr(ids, np.int32).copy()
    remap = np.zeros(len(r), np.int32)
    ref().ref_reorder(dim, P(arr(L)), cs, len(r), P(pos), P(r), P(ids), P(remap))
    return pos, r, ids, remap


def r_collisions(dim, L, cs, pos, r, ids=None):
    n = len(r)
    ids = np.arange(n, dtype=np.int32) if ids is None else ids
    per = np.zeros(n, np.uint8)
    anyc = ref().ref_collisions(dim, P(arr(L)), cs, n, P(arr(pos)), P(arr(r)), P(arr(ids, np.int32)), P(per))
    return bool(anyc), per


def r_rsa(dim, L, radii, max_attempts, seed):
    radii = arr(radii)
    n = len(radii)
    pos = np.zeros((n, dim))
    ids = np.zeros(n, np.int32)
    placed = np.zeros(1, np.int64)
    st = ref().ref_rsa_place(dim, P(arr(L)), n, P(radii), max_attempts, seed, P(pos), P(ids), P(placed))
    return st, pos, ids, int(placed[0])


def r_generate(dim, L, pos, r, ids, c_w, c_m, n_k, n_l, f_target, max_iterations, seed, reorder_period):
    pos = arr(pos).copy()
    r = arr(r).copy()
    ids = arr(ids, np.int32).copy()
    it = np.zeros(1, np.int64)
    f = np.zeros(1)
    acc = np.zeros(1, np.int64)
    st = ref().ref_generate(dim, P(arr(L)), len(r), P(pos), P(r), P(ids), c_w, c_m, n_k, n_l, f_target,
                            max_iterations, seed, reorder_period, P(it), P(f), P(acc))
    return st, pos, r, ids, int(it[0]), float(f[0]), int(acc[0])


def r_nnd(dim, L, pos):
    pos = arr(pos)
    out = np.zeros(len(pos))
    ref().ref_nnd(dim, P(arr(L)), len(pos), P(pos), P(out))
    return out


def r_histogram(values, bins, lo, hi):
    values = arr(values)
    counts = np.zeros(bins, np.int64)
    ref().ref_histogram(len(values), P(values), bins, lo, hi, P(counts))
    return counts


def r_bench_rounds(dim, L, pos, r, ids, c_m, n_l, rounds, seed, threads):
    acc = np.zeros(1, np.int64)
    secs = ref().ref_bench_rounds(dim, P(arr(L)), len(r), P(arr(pos)), P(arr(r)), P(arr(ids, np.int32)),
                                  c_m, n_l, rounds, seed, threads, P(acc))
    return secs, int(acc[0])


# ---- synthetic states ------------------------------------------------------------------
def random_particles(n, dim, rmin, rmax, L, seed):
    """fixtures.hpp:16-29 random_particles: uniform positions (random_point), radius
    uniform(rmin, rmax), drawn from the reference Rng through libsrm_ref."""
    u = np.zeros(n * (dim + 1))
    ref().ref_rng_uniforms(seed, len(u), P(u))
    u = u.reshape(n, dim + 1)
    pos = u[:, :dim] * np.asarray(L)[None, :]
    for a in range(dim):  # wrap (random.hpp:56-61)
        col = pos[:, a]
        col[col < 0.0] += L[a]
        col[col >= L[a]] -= L[a]
    r = rmin + (rmax - rmin) * u[:, dim]
    return np.ascontiguousarray(pos), np.ascontiguousarray(r)


# ---- platelets -------------------------------------------------------------------------
def o_pl_overlap(L, pa, na, Da, ta, pb, nb, Db, tb):
    return orc().orc_pl_overlap(P(arr(L)), P(arr(pa)), P(arr(na)), Da, ta, P(arr(pb)), P(arr(nb)), Db, tb)


def r_pl_overlap(L, pa, na, Da, ta, pb, nb, Db, tb):
    return ref().ref_pl_overlap(P(arr(L)), P(arr(pa)), P(arr(na)), Da, ta, P(arr(pb)), P(arr(nb)), Db, tb)


def o_pl_round(L, x0, n0, D, t, ids, slot, cell_size, c_m, c_r, n_l, seed, round_id, iteration):
    import math
    x0, n0 = arr(x0), arr(n0)
    n = len(D)
    xnew, nnew = np.zeros_like(x0), np.zeros_like(n0)
    acc = np.zeros(n, np.uint8)
    orc().orc_pl_sweep_round(P(arr(L)), n, P(x0), P(n0), P(arr(D)), P(arr(t)), P(arr(ids, np.int32)),
                             P(arr(slot, np.int32)), cell_size, c_m, math.cos(c_r), math.sin(c_r), n_l, seed,
                             round_id, iteration, P(xnew), P(nnew), P(acc))
    return xnew, nnew, acc


def o_pl_pairs(L, x, nrm, D, t, ids=None):
    n = len(D)
    ids = np.arange(n, dtype=np.int32) if ids is None else ids
    return orc().orc_pl_overlap_pairs(P(arr(L)), n, P(arr(x)), P(arr(nrm)), P(arr(D)), P(arr(t)),
                                      P(arr(ids, np.int32)))


def r_rsa_platelets(n, diameter, aspect, L, max_attempts, seed):
    pos = np.zeros((n, 3))
    nrm = np.zeros((n, 3))
    ids = np.zeros(n, np.int32)
    st = ref().ref_rsa_platelets(n, diameter, aspect, P(arr(L)), max_attempts, seed, P(pos), P(nrm), P(ids))
    return st, pos, nrm, ids


def r_local_nematic_order(L, pos, nrm, D, t, cutoff):
    """the reference's local_nematic_order (descriptors.hpp:182-209): (value, neighbor_count)"""
    n = len(D)
    value = np.zeros(n)
    count = np.zeros(n, np.int32)
    rc = ref().ref_local_nematic_order(P(arr(L)), n, P(arr(pos)), P(arr(nrm)), P(arr(D)), P(arr(t)), float(cutoff),
                                       P(value), P(count))
    if rc != 0:
        raise ValueError("local_nematic_order: cutoff must be positive")
    return value, count


def o_rsa_rounds(dim, L, radii, seed, max_rounds):
    """oracle/srm_oracle.c orc_rsa_rounds: (placed count, rounds, pos, placed flags)"""
    radii = arr(radii)
    n = len(radii)
    pos = np.zeros((n, dim))
    placed = np.zeros(n, np.uint8)
    rounds = C.c_int64()
    f = orc().orc_rsa_rounds
    f.restype = C.c_int64
    cnt = f(dim, P(arr(L)), n, P(radii), C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), int(max_rounds), P(pos), P(placed),
            C.byref(rounds))
    return cnt, rounds.value, pos, placed


def o_rsa_pl_rounds(L, n, D, aspect, seed, max_rounds):
    """oracle/srm_oracle.c orc_rsa_pl_rounds: (placed count, rounds, pos, normals, placed flags)"""
    pos = np.zeros((n, 3))
    nrm = np.zeros((n, 3))
    placed = np.zeros(n, np.uint8)
    rounds = C.c_int64()
    f = orc().orc_rsa_pl_rounds
    f.restype = C.c_int64
    f.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.c_double, C.c_uint64, C.c_int64, C.c_void_p, C.c_void_p,
                  C.c_void_p, C.c_void_p]
    cnt = f(P(arr(L)), n, D, D / aspect, C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), int(max_rounds), P(pos), P(nrm),
            P(placed), C.byref(rounds))
    return cnt, rounds.value, pos, nrm, placed
