"""Random sequential adsorption on the device:
bit for bit against the oracle's sequential restatement (orc_rsa_rounds) -- 2D/3D,
mono/polydisperse, dilute to dense -- and statistically against the reference's own
rsa_place (the same process with another random stream): per-seed NND summaries by
Welch t-tests across 10 configurations of 3000 spheres at f = 0.3."""
import numpy as np
import pytest

import orc
import paper_2605_18254_b200 as srm
import stats_util

pytestmark = pytest.mark.gpu


def _radii(dim, n, f, poly, seed):
    unit = np.pi if dim == 2 else 4.0 / 3.0 * np.pi
    r0 = (f / (n * unit)) ** (1.0 / dim)
    rng = np.random.default_rng(seed)
    return r0 * (rng.uniform(0.5, 1.5, n) if poly else np.ones(n))


@pytest.mark.parametrize("dim,n,f,poly,seed", [(3, 2000, 0.1, False, 1), (3, 1500, 0.3, False, 2),
                                               (2, 2500, 0.4, False, 3), (3, 1000, 0.15, True, 4),
                                               (2, 800, 0.2, True, 5)])
def test_rsa_device_bit_exact_vs_oracle(dim, n, f, poly, seed):
    L = [1.0] * dim
    r = _radii(dim, n, f, poly, seed)
    with srm.Context(L, n) as ctx:
        rounds = ctx.rsa_device(r, 0x1234 + seed)
        pos, rad, ids = ctx.download()
    cnt, orounds, opos, placed = orc.o_rsa_rounds(dim, L, r, 0x1234 + seed, 100000)
    assert cnt == n and placed.all() and rounds == orounds
    assert np.array_equal(ids, np.arange(n)) and np.array_equal(rad, r)
    assert np.array_equal(pos, opos)
    assert orc.o_stats(dim, L, pos, rad).overlap_pairs == 0


def test_rsa_device_placement_failure():
    r = _radii(3, 2000, 0.3, False, 9)
    with srm.Context([1.0] * 3, 2000) as ctx:
        with pytest.raises(srm.PlacementFailure):
            ctx.rsa_device(r, 7, max_rounds=2)


def test_rsa_device_statistics_match_reference_rsa():
    n, f, L = 3000, 0.3, [1.0, 1.0, 1.0]
    r = _radii(3, n, f, False, 0)
    rt = float(r[0])
    dev, ref = [], []
    for s in range(10):
        with srm.Context(L, n) as ctx:
            ctx.rsa_device(r, 100 + s)
            dev.append(ctx.nearest_neighbor_distances())
        st, pos, ids, _ = orc.r_rsa(3, L, r, 10000, 500 + s)
        assert st == 0
        ref.append(orc.r_nnd(3, L, pos))
    ps = stats_util.ensemble_agree(stats_util.ensemble_stats(dev, rt), stats_util.ensemble_stats(ref, rt))
    assert min(ps) > 1e-3, f"RSA NND summaries differ: Welch p = {ps}"
