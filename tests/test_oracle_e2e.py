"""The round semantics (coloured Gauss-Seidel sweep)
reproduce the reference's srm_generate statistically -- checked on the CPU with the
oracle's generate loop (orc.o_generate) against the reference ensembles in
tests/golden/e2e_*.npz, with the same tests the GPU end-to-end check applies."""
import os

import numpy as np
import pytest

import orc
import paper_2605_18254_b200 as srm
import stats_util

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("name", ["e2e_2d"])
def test_oracle_generate_statistics_match_reference(name):
    z = np.load(os.path.join(G, name + ".npz"))
    dim, n = int(z["dim"]), int(z["n"])
    L = [1.0] * dim
    unit = np.pi if dim == 2 else 4.0 / 3.0 * np.pi
    r0 = (float(z["f0"]) / (n * unit)) ** (1.0 / dim)
    nnd, rdf = [], []
    for s in z["seeds"]:
        pos, ids = srm.rsa_place(np.full(n, r0), L, 10000, 1000 + int(s))
        status, p, r, _, _, f, _ = orc.o_generate(dim, L, pos, np.full(n, r0), ids, float(z["c_w"]), float(z["c_m"]),
                                                  int(z["n_k"]), int(z["n_l"]), float(z["f_t"]), 100000, int(s))
        assert status == 0
        assert abs(f / float(z["f_t"]) - 1.0) < 1e-9
        assert orc.o_stats(dim, L, p, r).overlap_pairs == 0
        nnd.append(orc.r_nnd(dim, L, p))
        c = stats_util.rdf_counts(p, L, *stats_util.rdf_window(z))
        rdf.append(c)
    stats_util.check_against_reference(nnd, rdf, z)
