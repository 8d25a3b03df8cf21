"""Parity statistics on the device: nearest-neighbour distances
bit for bit against the reference's nearest_neighbor_distances (descriptors.hpp:96-115,
through oracle/_ref), its histogram (descriptors.hpp:254-277) bin for bin, and the
RDF pair counts against tests/stats_util.rdf_counts (numpy) count for count -- on dense
and sparse states, 2D and 3D, polydisperse, and grids small enough to force the ring
search to its all-particles fallback."""
import numpy as np
import pytest

import orc
import paper_2605_18254_b200 as srm
import stats_util

pytestmark = pytest.mark.gpu


def _state(dim, n, f, seed, poly=False):
    unit = np.pi if dim == 2 else 4.0 / 3.0 * np.pi
    r0 = (f / (n * unit)) ** (1.0 / dim)
    rng = np.random.default_rng(seed)
    r = r0 * (rng.uniform(0.6, 1.4, n) if poly else np.ones(n))
    L = [1.0] * dim
    pos, ids = srm.rsa_place(r, L, 100000, seed)
    return L, pos, r, ids


@pytest.mark.parametrize("dim,n,f,seed,poly", [(3, 5000, 0.30, 1, False), (3, 3000, 0.02, 2, False),
                                               (2, 4000, 0.45, 3, False), (2, 1500, 0.01, 4, True),
                                               (3, 4000, 0.25, 5, True), (3, 20, 0.001, 6, False)])
def test_nnd_and_histogram_bit_exact_vs_reference(dim, n, f, seed, poly):
    L, pos, r, ids = _state(dim, n, f, seed, poly)
    with srm.Context(L, n) as ctx:
        ctx.upload(pos, r, ids)
        d = ctx.nearest_neighbor_distances()
        ref = orc.r_nnd(dim, L, pos)
        assert np.array_equal(d, ref)
        lo, hi = float(np.quantile(ref, 0.05)), float(np.quantile(ref, 0.9))
        counts, total, inr = ctx.nnd_histogram(37, lo, hi)
    assert np.array_equal(counts, orc.r_histogram(ref, 37, lo, hi))
    assert total == n and inr == int(((ref >= lo) & (ref <= hi)).sum())


@pytest.mark.parametrize("dim,n,f,seed,poly,hi_rel", [(3, 4000, 0.30, 7, False, 5.0), (2, 3000, 0.4, 8, True, 6.0),
                                                      (3, 2000, 0.05, 9, False, 12.0), (3, 500, 0.2, 10, False, 40.0)])
def test_pair_counts_match_numpy(dim, n, f, seed, poly, hi_rel):
    L, pos, r, ids = _state(dim, n, f, seed, poly)
    rt = float(r.mean())
    lo, hi, bins = 2.0 * rt * 0.999, hi_rel * rt, 60
    with srm.Context(L, n) as ctx:
        ctx.upload(pos, r, ids)
        c = ctx.pair_counts(np.linspace(lo, hi, bins + 1))
    assert np.array_equal(c, stats_util.rdf_counts(pos, L, lo, hi, bins))


# ---- platelets (the platelet parity statistics on the device) -----------------
@pytest.mark.parametrize("n,aspect,rho,seed,cut_rel", [(3000, 20.0, 2.0, 11, 1.5), (800, 100.0, 3.0, 12, 1.0),
                                                        (200, 10.0, 1.0, 13, 4.0)])
def test_platelet_order_vs_reference(n, aspect, rho, seed, cut_rel):
    """local_nematic_order (descriptors.hpp:182-209): neighbour counts exact, values within
    1e-12 (the sum over neighbours runs in another cell order); centre NND bit for bit; the
    nearest-neighbour alignment and S2 against numpy."""
    box = 10.0
    L = [box] * 3
    D0 = (rho * box ** 3 / n) ** (1.0 / 3.0)
    st, pos, nrm, ids = orc.r_rsa_platelets(n, D0, aspect, L, 100000, seed)
    assert st == 0
    D, t = np.full(n, D0), np.full(n, D0 / aspect)
    cutoff = cut_rel * D0
    with srm.Context(L, n, shape="platelet") as ctx:
        ctx.upload_platelets(pos, nrm, D, t, ids)
        value, count = ctx.local_nematic_order(cutoff)
        nnd, align, s2 = ctx.platelet_summary()
        with pytest.raises(srm.ValidationError):
            ctx.local_nematic_order(0.0)
    v_ref, c_ref = orc.r_local_nematic_order(L, pos, nrm, D, t, cutoff)
    assert np.array_equal(count, c_ref)
    assert np.array_equal(np.isnan(value), np.isnan(v_ref))
    ok = ~np.isnan(v_ref)
    assert np.allclose(value[ok], v_ref[ok], rtol=1e-12, atol=0.0)
    assert np.array_equal(nnd, orc.r_nnd(3, L, pos))
    # nearest neighbour by brute force (ties have probability zero for random centres)
    d = pos[:, None, :] - pos[None, :, :]
    d -= box * np.round(d / box)
    d2 = (d * d).sum(-1)
    np.fill_diagonal(d2, np.inf)
    j = d2.argmin(1)
    assert np.allclose(align, np.abs((nrm * nrm[j]).sum(1)), rtol=0, atol=1e-14)
    Q = (3.0 * np.einsum("ni,nj->ij", nrm, nrm) / n - np.eye(3)) / 2.0
    assert abs(s2 - float(np.linalg.eigvalsh(Q)[-1])) < 1e-12
