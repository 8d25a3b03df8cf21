"""End-to-end parity on the GPU against the reference's own srm_generate (golden
ensembles in tests/golden/e2e_*.npz, produced by tests/golden/make_golden.py).

Same starts (rsa_place with the same seeds, bit-identical to the reference), same
parameters; the trajectories differ (parallel round vs sequential mt19937_64 sweep,
DESIGN.md §3), so the end states are compared statistically:
  * f_target reached within 1e-9 relative, zero overlaps (oracle audit);
  * nearest-neighbour-distance histogram (reference nearest_neighbor_distances), 40 bins
    over [2 r_t, 2.8 r_t] pooled over seeds: per-bin |dN| <= max(4 sigma, 2%), a chi-square
    homogeneity test and a two-sample KS test at alpha = 0.01 on the pooled samples;
  * RDF counts on [2 r_t, 5 r_t] (60 bins): per-bin |dN| <= max(4 sigma_Poisson, 2%), chi-square p > 0.01.
Also grid keys / reorder remap / collision flags on the golden states, bit-exact."""
import os

import numpy as np
import pytest

import orc
import paper_2605_18254_b200 as srm
import stats_util

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(G, name + ".npz"))


@pytest.mark.parametrize("name", ["grid_2d", "grid_3d"])
def test_device_grid_vs_golden(name):
    z = load(name)
    pos, r, L, cs = z["pos"], z["r"], list(z["L"]), float(z["cs"])
    with srm.Context(L, len(r)) as ctx:
        ctx.upload(pos, r)
        keys, order, _ = ctx.grid_build(cs)
        ctx.upload(pos, r)
        st = ctx.overlap_stats(2.5 * r.max())
    assert np.array_equal(keys.astype(np.uint64), z["keys"])
    assert np.array_equal(z["remap"][order], np.arange(len(r)))
    assert (st.overlap_pairs > 0) == bool(z["any"])


@pytest.mark.parametrize("name", ["e2e_2d", "e2e_3d"])
def test_generate_statistics_match_reference(name):
    z = load(name)
    dim, n = int(z["dim"]), int(z["n"])
    L = [1.0] * dim
    unit = np.pi if dim == 2 else 4.0 / 3.0 * np.pi
    r0 = (float(z["f0"]) / (n * unit)) ** (1.0 / dim)
    nnd, rdf = [], None
    for s in z["seeds"]:
        pos, ids = srm.rsa_place(np.full(n, r0), L, 10000, 1000 + int(s))
        snap = srm.Snapshot(L, pos, np.full(n, r0), ids)
        p = srm.SrmParams(c_w=float(z["c_w"]), c_m=float(z["c_m"]), n_k=int(z["n_k"]), n_l=int(z["n_l"]),
                          f_target=float(z["f_t"]), max_iterations=100000, seed=int(s), reorder_period=16)
        res = srm.srm_generate(snap, p)
        assert res.status == srm.GenerateStatus.Converged
        assert abs(res.snapshot.volume_fraction / float(z["f_t"]) - 1.0) < 1e-9
        out = res.snapshot
        assert orc.o_stats(dim, L, out.pos, out.radius).overlap_pairs == 0
        nnd.append(orc.r_nnd(dim, L, out.pos))
        c = stats_util.rdf_counts(out.pos, L, *stats_util.rdf_window(z))
        rdf = c if rdf is None else rdf + c
    stats_util.check_against_reference(nnd, rdf, z)
