"""Statistics for the end-to-end parity checks (test infrastructure).

rdf_counts: pair-distance histogram over [lo, hi) with the minimum image (the radial
distribution function up to its ideal-gas normalisation, which is identical for two
ensembles of equal N, box and bins).  The reference has no RDF; this one is
applied identically to the reference's and the B200 path's end states.
"""
import numpy as np


def rdf_counts(pos, L, lo, hi, bins):
    pos = np.asarray(pos, dtype=np.float64)
    L = np.asarray(L, dtype=np.float64)
    n = len(pos)
    counts = np.zeros(bins, np.int64)
    edges = np.linspace(lo, hi, bins + 1)
    step = 512
    for a in range(0, n, step):
        d = pos[a:a + step, None, :] - pos[None, :, :]
        d -= L * np.rint(d / L)
        r = np.sqrt((d * d).sum(-1))
        ii = np.arange(a, min(a + step, n))[:, None]
        jj = np.arange(n)[None, :]
        r = r[jj > ii]
        counts += np.histogram(r, bins=edges)[0]
    return counts


def hist_agree(c_a, c_b, rel=0.02, k=4.0):
    """per-bin agreement within max(k * sigma_Poisson, rel * count).
    k = 4: a family of 40-60 bins at 3 sigma alone false-alarms ~10% of the time on two
    samples of one distribution (seen: one NND bin at 3.3 sigma with KS p = 0.5); at 4
    sigma the family-wise rate is ~0.3%.  hist_chi2 is the whole-histogram test."""
    c_a = np.asarray(c_a, dtype=np.float64)
    c_b = np.asarray(c_b, dtype=np.float64)
    tol = np.maximum(k * np.sqrt(c_a + c_b + 1.0), rel * np.maximum(c_a, c_b))
    return np.abs(c_a - c_b) <= tol, tol


def hist_chi2(c_a, c_b):
    """two-sample chi-square homogeneity test of two histograms on the same bins
    (equal totals not required); returns the p-value."""
    from scipy import stats
    c_a = np.asarray(c_a, dtype=np.float64)
    c_b = np.asarray(c_b, dtype=np.float64)
    m = (c_a + c_b) > 0
    a, b = c_a[m], c_b[m]
    ka, kb = np.sqrt(b.sum() / a.sum()), np.sqrt(a.sum() / b.sum())
    chi2 = float((((ka * a - kb * b) ** 2) / (a + b)).sum())
    return float(stats.chi2.sf(chi2, m.sum() - 1))


def ensemble_stats(nnd_per_seed, scale, near=2.02):
    """Per-configuration summaries of nearest-neighbour distances (in units of `scale`):
    the 10/25/50/75/90% quantiles and, when `near` is given, the fraction below it."""
    rows = []
    for a in nnd_per_seed:
        a = np.asarray(a, dtype=np.float64) / scale
        row = list(np.quantile(a, [0.1, 0.25, 0.5, 0.75, 0.9]))
        if near is not None:
            row.append(float((a < near).mean()))
        rows.append(row)
    return np.array(rows)


def ensemble_agree(stats_a, stats_b, alpha=1e-3):
    """Welch t-test per summary statistic between two ensembles of configurations (one row
    per seed).  The pooled samples of one configuration are correlated, so a pooled
    two-sample KS test is miscalibrated: the reference against itself with other seeds
    gives KS p = 7e-12 at cfg 4 parameters (12 x 4000 spheres), while these per-seed tests
    give p = 0.01-0.6.  Returns the p-values; all must exceed alpha."""
    from scipy import stats
    return [float(stats.ttest_ind(stats_a[:, k], stats_b[:, k], equal_var=False).pvalue)
            for k in range(stats_a.shape[1])]


def ensemble_chi2(per_seed_a, per_seed_b):
    """Chi-square homogeneity of two ensembles of histograms (one row per configuration)
    with the between-configuration variance: sum over bins of (mean_a - mean_b)^2 /
    (se_a^2 + se_b^2).  Pooled Poisson chi-square treats the correlated samples of one
    configuration as independent (the reference against itself, other seeds: pooled
    p < 1e-6 at cfg 4 parameters); this one gives it 0.004-0.03.  Returns the p-value."""
    from scipy import stats
    a = np.asarray(per_seed_a, dtype=np.float64)
    b = np.asarray(per_seed_b, dtype=np.float64)
    va, vb = a.var(0, ddof=1) / len(a), b.var(0, ddof=1) / len(b)
    m = (va + vb) > 0
    c2 = float((((a.mean(0) - b.mean(0)) ** 2)[m] / (va + vb)[m]).sum())
    return float(stats.chi2.sf(c2, int(m.sum())))


def check_against_reference(nnd_list, rdf_list, z):
    """The e2e statistical parity of an ensemble of end states against the reference's
    (tests/golden/e2e_*.npz), at the level of configurations (one per seed): NND
    histograms (40 bins over [2 r_t, 2.8 r_t]) and RDF counts (60 bins over [2 r_t, 5 r_t])
    pooled per-bin within max(4 sigma, 2%) and by ensemble chi-square (p > 1e-3), and the
    per-seed NND summaries (quantiles, fraction within 1.01 contact) by Welch t-tests
    (ensemble_agree, p > 1e-3)."""
    rt = float(z["r_target"])
    bins = np.linspace(2.0 * rt * 0.999, 2.8 * rt, 41)
    h_dev = np.array([np.histogram(a, bins)[0] for a in nnd_list])
    h_ref = np.array([np.histogram(a, bins)[0] for a in z["nnd"]])
    ok, _ = hist_agree(h_dev.sum(0), h_ref.sum(0))
    assert ok.all(), f"NND bins out of tolerance: {np.where(~ok)[0]} dev={h_dev.sum(0)[~ok]} ref={h_ref.sum(0)[~ok]}"
    p = ensemble_chi2(h_dev, h_ref)
    assert p > 1e-3, f"NND histograms: ensemble chi2 p={p:.3g}"
    ps = ensemble_agree(ensemble_stats(nnd_list, rt), ensemble_stats(list(z["nnd"]), rt))
    assert min(ps) > 1e-3, f"per-seed NND summaries differ: Welch p = {ps}"
    rdf = np.sum(rdf_list, axis=0)
    ok, _ = hist_agree(rdf, z["rdf"])
    assert ok.all(), f"RDF bins out of tolerance: {np.where(~ok)[0]} dev={rdf[~ok]} ref={z['rdf'][~ok]}"
    p = ensemble_chi2(rdf_list, z["rdf_seeds"])
    assert p > 1e-3, f"RDF: ensemble chi2 p={p:.3g}"


def rdf_window(z):
    rt = float(z["r_target"])
    return 2.0 * rt * 0.999, 5.0 * rt, 60
