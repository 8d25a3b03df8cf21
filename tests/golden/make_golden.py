#!/usr/bin/env python
"""Generate the committed golden fixtures from the REFERENCE itself.

Run in the build container (needs oracle/_ref/libsrm_ref.so, built from the reference
sources by `make oracle`):   python tests/golden/make_golden.py

  grid_*.npz     seeded states + reference CellGrid::cell_of keys, reorder_by_locality
                 remap and per-particle check_particle_collision flags
  rsa_*.npz      reference rsa_place outputs (Rng(seed))
  e2e_*.npz      reference srm_generate end states for K seeds (f, iterations, nearest-
                 neighbour distances from the reference's nearest_neighbor_distances),
                 the statistical end-to-end oracle for tests/test_gpu_e2e.py; e2e_poly:
                 polydisperse, clustered starts (scaled-down cfg 3)
The reference ships no golden vectors of its own; these are produced by
its code and pinned here so the GPU box (which has no /root/reference) can use them.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import orc  # noqa: E402
import stats_util  # noqa: E402

# end-to-end statistical cases (scaled-down BASELINE configs)
E2E = {
    # name: dim, n, f0, f_target, c_m / r_target, c_w, n_k, n_l, seeds
    "e2e_2d": dict(dim=2, n=2000, f0=0.1, f_t=0.5, cm_rel=0.1, c_w=0.02, n_k=10, n_l=10, seeds=list(range(1, 17))),
    "e2e_3d": dict(dim=3, n=4000, f0=0.1, f_t=0.4, cm_rel=0.1, c_w=0.02, n_k=10, n_l=10, seeds=list(range(1, 13))),
    # the bench workload's parameters (cfg 4: f_t 0.30, c_m = 0.05 r_t): also the reference
    # side of the large-N spot check (tests/test_gpu_e2e.py, device NND / pair counts)
    "e2e_cfg4": dict(dim=3, n=4000, f0=0.1, f_t=0.3, cm_rel=0.05, c_w=0.02, n_k=10, n_l=10, seeds=list(range(1, 13))),
}


def unit(dim):
    return np.pi if dim == 2 else 4.0 / 3.0 * np.pi


def e2e_case(name, c):
    dim, n = c["dim"], c["n"]
    L = [1.0] * dim
    r0 = (c["f0"] / (n * unit(dim))) ** (1.0 / dim)
    rt = (c["f_t"] / (n * unit(dim))) ** (1.0 / dim)
    c_m = c["cm_rel"] * rt
    nnd, fs, its, accs, rdf, rdf_seeds = [], [], [], [], None, []
    for s in c["seeds"]:
        st, pos, ids, _ = orc.r_rsa(dim, L, np.full(n, r0), 10000, 1000 + s)
        assert st == 0
        st, pos, r, ids, it, f, acc = orc.r_generate(dim, L, pos, np.full(n, r0), ids, c["c_w"], c_m, c["n_k"],
                                                     c["n_l"], c["f_t"], 100000, s, 16)
        assert st == 0, f"reference srm_generate did not converge ({name}, seed {s})"
        nnd.append(orc.r_nnd(dim, L, pos))
        c_rdf = stats_util.rdf_counts(pos, L, 2.0 * rt * 0.999, 5.0 * rt, 60)
        rdf = c_rdf if rdf is None else rdf + c_rdf
        rdf_seeds.append(c_rdf)
        fs.append(f)
        its.append(it)
        accs.append(acc)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), nnd=np.array(nnd), f=np.array(fs),
                        iterations=np.array(its), accepted=np.array(accs), r_target=rt, c_m=c_m, rdf=rdf,
                        rdf_seeds=np.array(rdf_seeds),
                        **{k: np.array(v) for k, v in c.items()})
    print(name, "iterations", its, "f", fs[0])


# scaled-down cfg 3: polydisperse lognormal radii (mean 1, CV 0.2, clipped to [0.5, 2]),
# clustered start (the package's rsa_clustered, deterministic, so the GPU test rebuilds
# the same starts), f 0.05 -> 0.45, c_m = 0.1
POLY = dict(n=2000, f0=0.05, f_t=0.45, c_m=0.1, c_w=0.02, n_k=10, n_l=10, clusters=20, sigma=3.0,
            seeds=list(range(1, 13)))


def poly_start(c, seed):
    import math
    import paper_2605_18254_b200 as srm
    s2 = math.log(1.04)
    rng = np.random.default_rng(seed)
    r_t = np.clip(rng.lognormal(-0.5 * s2, math.sqrt(s2), c["n"]), 0.5, 2.0)
    L = float((np.sum(4.0 / 3.0 * np.pi * r_t ** 3) / c["f_t"]) ** (1.0 / 3.0))
    r0 = r_t * (c["f0"] / c["f_t"]) ** (1.0 / 3.0)
    pos, ids = srm.rsa_clustered(r0, [L] * 3, c["clusters"], c["sigma"], 10000, 100 + seed)
    return [L] * 3, pos, r0, ids


def e2e_poly_case(name, c):
    nnd, rdf, its, rdf_seeds = [], None, [], []
    for s in c["seeds"]:
        L, pos, r0, ids = poly_start(c, s)
        st, pos, r, ids, it, f, acc = orc.r_generate(3, L, pos, r0, ids, c["c_w"], c["c_m"], c["n_k"], c["n_l"],
                                                     c["f_t"], 100000, s, 16)
        assert st == 0, f"reference srm_generate did not converge ({name}, seed {s})"
        rm = float(r.mean())
        nnd.append(orc.r_nnd(3, L, pos) / rm)
        c_rdf = stats_util.rdf_counts(pos / rm, np.array(L) / rm, 0.9 * 2, 5.0 * 2, 60)  # in units of mean r
        rdf = c_rdf if rdf is None else rdf + c_rdf
        rdf_seeds.append(c_rdf)
        its.append(it)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), nnd=np.array(nnd), rdf=rdf, iterations=np.array(its),
                        rdf_seeds=np.array(rdf_seeds),
                        **{k: np.array(v) for k, v in c.items()})
    print(name, "iterations", its)


# the reference at the spot check's size (one 10^6-sphere run at cfg 4 parameters): its
# NND summaries and histogram (reference nearest_neighbor_distances) and pair counts
# (scipy cKDTree, periodic) -- the state itself (24 MB) is not kept
LARGE = dict(dim=3, n=1_000_000, f0=0.1, f_t=0.3, cm_rel=0.05, c_w=0.02, n_k=10, n_l=10, seeds=[1])


def e2e_large_case(name, c):
    from scipy.spatial import cKDTree
    n = c["n"]
    L = [1.0] * 3
    r0 = (c["f0"] / (n * unit(3))) ** (1.0 / 3.0)
    rt = (c["f_t"] / (n * unit(3))) ** (1.0 / 3.0)
    out = {}
    for s in c["seeds"]:
        st, pos, ids, _ = orc.r_rsa(3, L, np.full(n, r0), 10000, 1000 + s)
        assert st == 0
        st, pos, r, ids, it, f, acc = orc.r_generate(3, L, pos, np.full(n, r0), ids, c["c_w"], c["cm_rel"] * rt,
                                                     c["n_k"], c["n_l"], c["f_t"], 100000, s, 16)
        assert st == 0
        nnd = orc.r_nnd(3, L, pos) / rt
        out["summary"] = stats_util.ensemble_stats([nnd], 1.0)[0]
        out["nnd_hist"] = np.histogram(nnd, np.linspace(2.0 * 0.999, 2.8, 41))[0]
        edges = np.linspace(2.0 * 0.999, 5.0, 61) * rt
        cum = cKDTree(pos, boxsize=1.0).count_neighbors(cKDTree(pos, boxsize=1.0), edges)
        out["rdf"] = np.diff(cum) // 2  # ordered pairs -> unordered
        out["iterations"] = it
    np.savez_compressed(os.path.join(HERE, name + ".npz"), r_target=rt, **out, **{k: np.array(v) for k, v in c.items()})
    print(name, out["summary"], out["iterations"])


# scaled-down cfg 5: thin platelets (aspect 20), reference rsa_platelets start (D = 1,
# box 7: rho = 1.17), grown to f = 0.14 (D ~ 1.46) with c_w 0.01, c_m = c_r = 0.05
PLATE = dict(n=400, L=7.0, aspect=20.0, c_w=0.01, c_m=0.05, c_r=0.05, n_k=10, n_l=10, f_t=0.14,
             seeds=list(range(1, 17)))


def platelet_stats(pos, nrm, D, L):
    """Per-configuration summaries of a platelet packing: centre NND quantiles in units of
    D, the nematic order S2 (largest eigenvalue of <(3 n n - 1) / 2>), the mean |n . n'|
    of nearest-neighbour pairs, and the fraction of centres closer than D / 2."""
    nnd = orc.r_nnd(3, L, pos) / D
    q = np.quantile(nnd, [0.1, 0.25, 0.5, 0.75, 0.9])
    Q = (3.0 * np.einsum("ni,nj->ij", nrm, nrm) / len(nrm) - np.eye(3)) / 2.0
    s2 = float(np.linalg.eigvalsh(Q)[-1])
    from scipy.spatial import cKDTree
    t = cKDTree(pos, boxsize=L[0])
    _, j = t.query(pos, k=2)
    align = float(np.abs(np.einsum("ni,ni->n", nrm, nrm[j[:, 1]])).mean())
    close = float((nnd < 0.5).mean())
    return np.concatenate([q, [s2, align, close]]), nnd


def e2e_platelet_case(name, c):
    import ctypes as C
    stats, nnds = [], []
    L = [c["L"]] * 3
    for s in c["seeds"]:
        st, pos, nrm, ids = orc.r_rsa_platelets(c["n"], 1.0, c["aspect"], L, 10000, 100 + s)
        assert st == 0
        D = np.full(c["n"], 1.0)
        th = D / c["aspect"]
        it = np.zeros(1, np.int64)
        f = np.zeros(1)
        P = orc.P
        rc = orc.ref().ref_generate_platelets(P(orc.arr(L)), c["n"], P(pos), P(nrm), P(D), P(th), P(ids), c["c_w"],
                                              c["c_m"], c["c_r"], c["n_k"], c["n_l"], c["f_t"], 100000, s, 16,
                                              P(it), P(f))
        assert rc == 0, f"reference platelet srm_generate did not converge (seed {s})"
        row, nnd = platelet_stats(pos, nrm, float(D[0]), L)
        stats.append(row)
        nnds.append(nnd)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), stats=np.array(stats), nnd=np.array(nnds),
                        **{k: np.array(v) for k, v in c.items()})
    print(name, np.array(stats).mean(0))


# cfg 4's parameters at N = 10^6, an ensemble of reference runs (the spot check's
# tolerance is the reference's own configuration-to-configuration spread AT this N)
LARGE_ENS = dict(n=1_000_000, f0=0.1, f_t=0.3, cm_rel=0.05, c_w=0.02, n_k=10, n_l=10, seeds=[1, 2, 3, 4])


def _large_one(args):
    c, s = args
    from scipy.spatial import cKDTree
    n = c["n"]
    L = [1.0] * 3
    r0 = (c["f0"] / (n * unit(3))) ** (1.0 / 3.0)
    rt = (c["f_t"] / (n * unit(3))) ** (1.0 / 3.0)
    st, pos, ids, _ = orc.r_rsa(3, L, np.full(n, r0), 10000, 1000 + s)
    assert st == 0
    st, pos, r, ids, it, f, acc = orc.r_generate(3, L, pos, np.full(n, r0), ids, c["c_w"], c["cm_rel"] * rt,
                                                 c["n_k"], c["n_l"], c["f_t"], 100000, s, 16)
    assert st == 0
    nnd = orc.r_nnd(3, L, pos) / rt
    edges = np.linspace(2.0 * 0.999, 5.0, 61) * rt
    cum = cKDTree(pos, boxsize=1.0).count_neighbors(cKDTree(pos, boxsize=1.0), edges)
    return (stats_util.ensemble_stats([nnd], 1.0)[0], np.histogram(nnd, np.linspace(2.0 * 0.999, 2.8, 41))[0],
            np.diff(cum) // 2, it)


def e2e_large_ensemble(name, c):
    from multiprocessing import Pool
    with Pool(len(c["seeds"])) as pool:
        res = pool.map(_large_one, [(c, s) for s in c["seeds"]])
    rt = (c["f_t"] / (c["n"] * unit(3))) ** (1.0 / 3.0)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), r_target=rt, summary=np.array([r[0] for r in res]),
                        nnd_hist=np.array([r[1] for r in res]), rdf=np.array([r[2] for r in res]),
                        iterations=np.array([r[3] for r in res]), **{k: np.array(v) for k, v in c.items()})
    print(name, np.array([r[0] for r in res]), [r[3] for r in res])


# cfg 1 at full size with BASELINE's literal start: uniform random centres (numpy PCG64,
# seed 5000 + s), radius grown from half the smallest centre distance (reference
# nearest_neighbor_distances) x (1 - 1e-9) to f = 0.5; c_m = 0.1 r_t, c_w 0.02, n_k = n_l = 10
CFG1 = dict(n=10_000, f_t=0.5, cm_rel=0.1, c_w=0.02, n_k=10, n_l=10, seeds=list(range(1, 13)))


def cfg1_start(n, s):
    pos = np.random.default_rng(5000 + s).random((n, 2))
    return pos


def e2e_cfg1_full(name, c):
    n = c["n"]
    L = [1.0, 1.0]
    rt = (c["f_t"] / (n * np.pi)) ** 0.5
    nnd, r0s, its, rdf_seeds = [], [], [], []
    for s in c["seeds"]:
        pos = cfg1_start(n, s)
        r0 = 0.5 * float(orc.r_nnd(2, L, pos).min()) * (1.0 - 1e-9)
        st, pos, r, ids, it, f, acc = orc.r_generate(2, L, pos, np.full(n, r0), np.arange(n, dtype=np.int32),
                                                     c["c_w"], c["cm_rel"] * rt, c["n_k"], c["n_l"], c["f_t"],
                                                     100000, s, 16)
        assert st == 0
        nnd.append(orc.r_nnd(2, L, pos))
        rdf_seeds.append(stats_util.rdf_counts(pos, L, 2.0 * rt * 0.999, 5.0 * rt, 60))
        r0s.append(r0)
        its.append(it)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), nnd=np.array(nnd), r0=np.array(r0s),
                        iterations=np.array(its), r_target=rt, c_m=c["cm_rel"] * rt, rdf=np.sum(rdf_seeds, 0),
                        rdf_seeds=np.array(rdf_seeds), dim=2, f0=0.0, **{k: np.array(v) for k, v in c.items()})
    print(name, its, r0s[:3])


def grid_case(name, dim, n, rmin, rmax, cs, seed, L):
    pos, r = orc.random_particles(n, dim, rmin, rmax, L, seed)
    keys, _ = orc.r_keys(dim, L, cs, pos)
    _, _, _, remap = orc.r_reorder(dim, L, cs, pos, r, np.arange(n, dtype=np.int32))
    anyc, per = orc.r_collisions(dim, L, cs, pos, r)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), pos=pos, r=r, L=np.array(L), cs=cs, keys=keys,
                        remap=remap, per=per, any=anyc)


def rsa_case(name, dim, n, f, seed):
    L = [1.0] * dim
    r = (f / (n * unit(dim))) ** (1.0 / dim)
    st, pos, ids, _ = orc.r_rsa(dim, L, np.full(n, r), 10000, seed)
    assert st == 0
    np.savez_compressed(os.path.join(HERE, name + ".npz"), pos=pos, ids=ids, r=r, seed=seed, L=np.array(L))


def main():
    if len(sys.argv) > 1:  # named cases only
        for name in sys.argv[1:]:
            if name == "e2e_poly":
                e2e_poly_case(name, POLY)
            elif name == "e2e_cfg4_large":
                e2e_large_case(name, LARGE)
            elif name == "e2e_cfg4_large_ens":
                e2e_large_ensemble(name, LARGE_ENS)
            elif name == "e2e_cfg1_full":
                e2e_cfg1_full(name, CFG1)
            elif name == "e2e_platelet":
                e2e_platelet_case(name, PLATE)
            else:
                e2e_case(name, E2E[name])
        return
    grid_case("grid_2d", 2, 3000, 0.001, 0.004, 0.012, 11, [1.0, 1.0])
    grid_case("grid_3d", 3, 4000, 0.004, 0.02, 0.05, 12, [1.0, 1.3, 0.8])
    rsa_case("rsa_2d", 2, 800, 0.4, 5)
    rsa_case("rsa_3d", 3, 800, 0.25, 6)
    for name, c in E2E.items():
        e2e_case(name, c)
    e2e_poly_case("e2e_poly", POLY)
    e2e_platelet_case("e2e_platelet", PLATE)


if __name__ == "__main__":
    main()
