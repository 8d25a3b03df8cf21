"""The device-resident srm_generate (one CUDA graph with conditional nodes, DESIGN.md
§3.4) against the host-driven loop over the same kernels: identical decisions and
identical end states when no clamped final swell is involved (budget-limited runs), the
same convergence otherwise (the clamp factor's pow is the device's, 1 ulp at most from
glibc's).  Also the reorder cadence, shake rounds and progress records through the graph."""
import numpy as np
import pytest

import orc
import paper_2605_18254_b200 as srm

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["", "lane", "trials", "wave", "resolve"])
def sweep_kernel(request, monkeypatch):
    """Every test once per sweep kernel (SRM_B200_SWEEP: "" = chosen by the grid, lane =
    k_sweep_warpq, trials = k_sweep_trials, team = k_sweep_team, wave = the one-launch wavefront
    k_sweep_wave where the grid allows it): each is exact on any grid."""
    if request.param:
        monkeypatch.setenv("SRM_B200_SWEEP", request.param)
    else:
        monkeypatch.delenv("SRM_B200_SWEEP", raising=False)
    return request.param


def _start(dim, n, f0, seed, poly=False):
    rng = np.random.default_rng(seed)
    unit = np.pi if dim == 2 else 4.0 / 3.0 * np.pi
    r0 = (f0 / (n * unit)) ** (1.0 / dim)
    radii = np.full(n, r0) if not poly else r0 * rng.uniform(0.7, 1.2, n)
    if poly == "bi":  # 1 in 20 four times larger: crowded cells (the team sweep)
        rel = np.ones(n)
        rel[: n // 20] = 4.0
        radii = rel * (f0 / (unit * np.sum(rel ** dim))) ** (1.0 / dim)
    L = [1.0] * dim
    pos, ids = srm.rsa_place(radii, L, srm.K_RSA_DEFAULT_ATTEMPTS, seed)
    return L, pos, radii, ids


def _run(L, pos, r, ids, params, device_loop, it0=0):
    recs = []
    with srm.Context(L, len(r)) as ctx:
        ctx.upload(pos, r, ids)
        ctx.set_generate_mode(device_loop)
        out = ctx.generate(params, it0, progress=recs.append)
        p, rr, i = ctx.download()
    return out, p, rr, i, recs


@pytest.mark.parametrize("dim,n,f0,poly,reorder", [(2, 3000, 0.2, False, 4), (3, 6000, 0.15, False, 3),
                                                    (3, 4000, 0.12, True, 0), (3, 12000, 0.15, "bi", 3)])
def test_budget_limited_runs_are_identical(dim, n, f0, poly, reorder):
    L, pos, r, ids = _start(dim, n, f0, 11, poly)
    c_m = 0.1 * float(r.max())
    # c_w large enough that rounds fail now and then (shake rounds), budget before f_t
    p = srm.SrmParams(c_w=0.08, c_m=c_m, n_k=3, n_l=6, f_target=0.6 if dim == 2 else 0.45, max_iterations=12,
                      seed=99, reorder_period=reorder)
    a = _run(L, pos, r, ids, p, device_loop=False, it0=5)
    b = _run(L, pos, r, ids, p, device_loop=True, it0=5)
    oa, ob = a[0], b[0]
    assert oa.status == ob.status == 1  # IterationLimitExceeded
    for k in ("iteration_count", "accepted_iterations", "rounds", "shake_rounds"):
        assert getattr(oa, k) == getattr(ob, k), k
    assert oa.volume_fraction == ob.volume_fraction
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])
    # progress: the same records (elapsed times aside)
    assert [(x.iteration, x.volume_fraction, x.accepted, x.rounds) for x in a[4]] == \
           [(x.iteration, x.volume_fraction, x.accepted, x.rounds) for x in b[4]]
    assert len(b[4]) == 12 and b[4][0].iteration == 6


@pytest.mark.parametrize("dim,n,ft", [(2, 2000, 0.5), (3, 4000, 0.35)])
def test_converged_runs_agree(dim, n, ft):
    L, pos, r, ids = _start(dim, n, 0.1, 5)
    p = srm.SrmParams(c_w=0.02, c_m=0.1 * float(r.max()) * (ft / 0.1) ** (1.0 / dim), n_k=10, n_l=10, f_target=ft,
                      seed=3, reorder_period=16)
    a = _run(L, pos, r, ids, p, device_loop=False)
    b = _run(L, pos, r, ids, p, device_loop=True)
    for o, pp, rr in ((a[0], a[1], a[2]), (b[0], b[1], b[2])):
        assert o.status == 0
        assert abs(o.volume_fraction / ft - 1.0) < 1e-12
        assert orc.o_stats(dim, L, pp, rr).overlap_pairs == 0
    assert abs(a[0].iteration_count - b[0].iteration_count) <= 1
