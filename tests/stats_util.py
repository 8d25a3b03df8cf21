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


def check_against_reference(nnd_list, rdf, z):
    """The e2e statistical parity of an ensemble of end states against the reference's
    (tests/golden/e2e_*.npz): NND histogram (40 bins over [2 r_t, 2.8 r_t]) per-bin and
    chi-square, two-sample KS on the pooled NND samples, RDF counts per-bin and chi-square."""
    from scipy import stats
    rt = float(z["r_target"])
    nnd = np.concatenate(nnd_list)
    ref = z["nnd"].ravel()
    bins = np.linspace(2.0 * rt * 0.999, 2.8 * rt, 41)
    h_dev = np.histogram(nnd, bins)[0]
    h_ref = np.histogram(ref, bins)[0]
    ok, _ = hist_agree(h_dev, h_ref)
    assert ok.all(), f"NND bins out of tolerance: {np.where(~ok)[0]} dev={h_dev[~ok]} ref={h_ref[~ok]}"
    p = hist_chi2(h_dev, h_ref)
    assert p > 0.01, f"NND histogram chi2 p={p:.3g}"
    ks = stats.ks_2samp(nnd, ref)
    assert ks.pvalue > 0.01, f"KS p={ks.pvalue:.3g} stat={ks.statistic:.4f}"
    ok, _ = hist_agree(rdf, z["rdf"])
    assert ok.all(), f"RDF bins out of tolerance: {np.where(~ok)[0]} dev={rdf[~ok]} ref={z['rdf'][~ok]}"
    p = hist_chi2(rdf, z["rdf"])
    assert p > 0.01, f"RDF chi2 p={p:.3g}"


def rdf_window(z):
    rt = float(z["r_target"])
    return 2.0 * rt * 0.999, 5.0 * rt, 60
