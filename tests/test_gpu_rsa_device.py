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


# ---- platelets: rsa_platelets (recipes.cpp:107-148) in rounds ---------------------------
@pytest.mark.parametrize("n,L,aspect,seed", [(300, 6.0, 20.0, 5), (500, 8.0, 100.0, 6), (2000, 12.0, 100.0, 7)])
def test_rsa_platelets_device_bit_exact_vs_oracle(n, L, aspect, seed):
    Lb = [L] * 3
    with srm.Context(Lb, n, shape="platelet") as ctx:
        rounds = ctx.rsa_platelets_device(n, 1.0, aspect, 0x77 + seed)
        pos, nrm, D, t, ids = ctx.download_platelets()
    cnt, orounds, opos, onrm, placed = orc.o_rsa_pl_rounds(Lb, n, 1.0, aspect, 0x77 + seed, 100000)
    assert cnt == n and placed.all() and rounds == orounds
    assert np.array_equal(ids, np.arange(n))
    assert np.array_equal(pos, opos) and np.array_equal(nrm, onrm)
    assert np.all(D == 1.0) and np.all(t == 1.0 / aspect)
    assert orc.o_pl_pairs(Lb, pos, nrm, D, t, ids) == 0  # no ordered pair overlaps


def test_rsa_platelets_device_statistics_match_reference():
    """The same process as the reference's rsa_platelets with another random stream:
    per-seed centre-NND quantiles and the nematic order parameter (isotropic start) by
    Welch t-tests across 12 configurations of 1500 platelets (aspect 20, rho = 2)."""
    n, aspect = 1500, 20.0
    L = (n / 2.0) ** (1.0 / 3.0)
    Lb = [L] * 3

    def summary(pos, nrm):
        nnd = orc.r_nnd(3, Lb, pos)
        q = np.quantile(nnd, [0.1, 0.25, 0.5, 0.75, 0.9])
        Q = 1.5 * (nrm[:, :, None] * nrm[:, None, :]).mean(0) - 0.5 * np.eye(3)
        return np.concatenate([q, [np.linalg.eigvalsh(Q).max()]])

    dev, ref = [], []
    for s in range(12):
        with srm.Context(Lb, n, shape="platelet") as ctx:
            ctx.rsa_platelets_device(n, 1.0, aspect, 900 + s)
            pos, nrm, _, _, _ = ctx.download_platelets()
        dev.append(summary(pos, nrm))
        st, rpos, rnrm, _ = orc.r_rsa_platelets(n, 1.0, aspect, Lb, 100000, 900 + s)
        assert st == 0
        ref.append(summary(rpos, rnrm))
    ps = stats_util.ensemble_agree(np.array(dev), np.array(ref))
    assert min(ps) > 1e-3, f"device vs reference rsa_platelets summaries: Welch p = {ps}"


def test_rsa_platelets_device_errors():
    with srm.Context([5.0] * 3, 10, shape="platelet") as ctx:
        with pytest.raises(srm.ValidationError):
            ctx.rsa_platelets_device(10, 1.0, 1.0, 1)  # aspect ratio must exceed 1
        with pytest.raises(srm.ValidationError):
            ctx.rsa_platelets_device(10, 2.5, 20.0, 1)  # too large for the box (bound 1.31 > 5 / 4)
        with pytest.raises(srm.PlacementFailure):
            ctx.rsa_platelets_device(10, 1.2, 20.0, 1, max_rounds=1)
    with srm.Context([5.0] * 3, 10) as sph:
        with pytest.raises(srm.ValidationError):
            sph.rsa_platelets_device(10, 1.0, 20.0, 1)
