#!/usr/bin/env python
"""Generate the committed golden fixtures from the REFERENCE itself.

Run in the build container (needs oracle/_ref/libsrm_ref.so, built from the reference
sources by `make oracle`):   python tests/golden/make_golden.py

  grid_*.npz     seeded states + reference CellGrid::cell_of keys, reorder_by_locality
                 remap and per-particle check_particle_collision flags
  rsa_*.npz      reference rsa_place outputs (Rng(seed))
  e2e_*.npz      reference srm_generate end states for K seeds (f, iterations, nearest-
                 neighbour distances from the reference's nearest_neighbor_distances),
                 the statistical end-to-end oracle for tests/test_gpu_e2e.py
The reference ships no golden vectors of its own; these are produced by
its code and pinned here so the GPU box (which has no /root/reference) can use them.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import orc  # noqa: E402
import stats_util  # noqa: E402

# end-to-end statistical cases (scaled-down BASELINE configs)
E2E = {
    # name: dim, n, f0, f_target, c_m / r_target, c_w, n_k, n_l, seeds
    "e2e_2d": dict(dim=2, n=2000, f0=0.1, f_t=0.5, cm_rel=0.1, c_w=0.02, n_k=10, n_l=10, seeds=list(range(1, 17))),
    "e2e_3d": dict(dim=3, n=4000, f0=0.1, f_t=0.4, cm_rel=0.1, c_w=0.02, n_k=10, n_l=10, seeds=list(range(1, 13))),
}


def unit(dim):
    return np.pi if dim == 2 else 4.0 / 3.0 * np.pi


def e2e_case(name, c):
    dim, n = c["dim"], c["n"]
    L = [1.0] * dim
    r0 = (c["f0"] / (n * unit(dim))) ** (1.0 / dim)
    rt = (c["f_t"] / (n * unit(dim))) ** (1.0 / dim)
    c_m = c["cm_rel"] * rt
    nnd, fs, its, accs, rdf = [], [], [], [], None
    for s in c["seeds"]:
        st, pos, ids, _ = orc.r_rsa(dim, L, np.full(n, r0), 10000, 1000 + s)
        assert st == 0
        st, pos, r, ids, it, f, acc = orc.r_generate(dim, L, pos, np.full(n, r0), ids, c["c_w"], c_m, c["n_k"],
                                                     c["n_l"], c["f_t"], 100000, s, 16)
        assert st == 0, f"reference srm_generate did not converge ({name}, seed {s})"
        nnd.append(orc.r_nnd(dim, L, pos))
        c_rdf = stats_util.rdf_counts(pos, L, 2.0 * rt * 0.999, 5.0 * rt, 60)
        rdf = c_rdf if rdf is None else rdf + c_rdf
        fs.append(f)
        its.append(it)
        accs.append(acc)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), nnd=np.array(nnd), f=np.array(fs),
                        iterations=np.array(its), accepted=np.array(accs), r_target=rt, c_m=c_m, rdf=rdf,
                        **{k: np.array(v) for k, v in c.items()})
    print(name, "iterations", its, "f", fs[0])


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
    grid_case("grid_2d", 2, 3000, 0.001, 0.004, 0.012, 11, [1.0, 1.0])
    grid_case("grid_3d", 3, 4000, 0.004, 0.02, 0.05, 12, [1.0, 1.3, 0.8])
    rsa_case("rsa_2d", 2, 800, 0.4, 5)
    rsa_case("rsa_3d", 3, 800, 0.25, 6)
    for name, c in E2E.items():
        e2e_case(name, c)


if __name__ == "__main__":
    main()
