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


def hist_agree(c_a, c_b, rel=0.02, k=3.0):
    """per-bin agreement within max(k * sigma_Poisson, rel * count)."""
    c_a = np.asarray(c_a, dtype=np.float64)
    c_b = np.asarray(c_b, dtype=np.float64)
    tol = np.maximum(k * np.sqrt(c_a + c_b + 1.0), rel * np.maximum(c_a, c_b))
    return np.abs(c_a - c_b) <= tol, tol
