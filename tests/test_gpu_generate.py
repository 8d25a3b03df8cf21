"""srm_generate and friends on the GPU: the engine-level cases of the reference's
test_engine.cpp (convergence, validity, budget, progress, validation, determinism),
re-expressed against the B200 path.  Validity uses the oracle's all-pairs audit."""
import numpy as np
import pytest

import orc
import paper_2605_18254_b200 as srm

pytestmark = pytest.mark.gpu


def disk_start(n, f0, seed):
    # test_engine.cpp:15-23
    r = np.sqrt(f0 / (n * np.pi))
    pos, ids = srm.rsa_place(np.full(n, r), [1.0, 1.0], srm.K_RSA_DEFAULT_ATTEMPTS, seed)
    s = srm.Snapshot([1.0, 1.0], pos, np.full(n, r), ids)
    s.refresh_volume_fraction()
    return s


def violations(snap, rel_tol):
    """oracles.hpp:41-52 sphere_overlap_violations via brute force numpy"""
    L = np.asarray(snap.box)
    d = snap.pos[:, None, :] - snap.pos[None, :, :]
    d -= L * np.rint(d / L)
    dist = np.sqrt((d * d).sum(-1))
    rr = snap.radius[:, None] + snap.radius[None, :]
    bad = dist < rr * (1.0 - rel_tol)
    np.fill_diagonal(bad, False)
    return int(bad.sum() // 2)


def test_generate_reaches_target_2d():
    snap = disk_start(100, 0.1, 42)
    p = srm.SrmParams(c_w=0.05, c_m=0.01, n_k=8, n_l=8, f_target=0.5, seed=7)
    res = srm.srm_generate(snap, p)
    assert res.status == srm.GenerateStatus.Converged
    assert 0.5 * (1 - 1e-12) <= res.snapshot.volume_fraction <= 0.5 * (1 + 1e-9)
    assert violations(res.snapshot, 1e-12) == 0
    assert orc.o_stats(2, [1, 1], res.snapshot.pos, res.snapshot.radius).overlap_pairs == 0
    assert res.snapshot.iteration_count > 0
    res.snapshot.refresh_volume_fraction()
    assert res.snapshot.volume_fraction == pytest.approx(0.5, rel=1e-12)


def test_generate_3d():
    r = np.cbrt(0.05 * 3.0 / (100 * 4.0 * np.pi))
    pos, ids = srm.rsa_place(np.full(100, r), [1, 1, 1], srm.K_RSA_DEFAULT_ATTEMPTS, 11)
    snap = srm.Snapshot([1, 1, 1], pos, np.full(100, r), ids)
    res = srm.srm_generate(snap, srm.SrmParams(c_w=0.05, c_m=0.02, f_target=0.3, seed=3))
    assert res.status == srm.GenerateStatus.Converged
    assert res.snapshot.volume_fraction >= 0.3 * (1 - 1e-12)
    assert violations(res.snapshot, 1e-12) == 0


def test_already_at_target_returns_input():
    snap = disk_start(100, 0.2, 6)
    res = srm.srm_generate(snap, srm.SrmParams(c_w=0.05, f_target=0.15))
    assert res.status == srm.GenerateStatus.Converged
    assert np.array_equal(res.snapshot.pos, snap.pos) and np.array_equal(res.snapshot.radius, snap.radius)
    assert res.snapshot.iteration_count == snap.iteration_count


def test_deterministic_under_seed():
    snap = disk_start(80, 0.1, 9)
    p = srm.SrmParams(c_w=0.05, c_m=0.01, f_target=0.4, seed=31)
    a = srm.srm_generate(snap, p)
    b = srm.srm_generate(snap, p)
    assert np.array_equal(a.snapshot.pos, b.snapshot.pos)
    p.seed = 32
    c = srm.srm_generate(snap, p)
    assert not np.array_equal(a.snapshot.pos, c.snapshot.pos)


def test_iteration_budget():
    snap = disk_start(100, 0.1, 12)
    res = srm.srm_generate(snap, srm.SrmParams(c_w=0.001, c_m=0.01, f_target=0.5, max_iterations=5))
    assert res.status == srm.GenerateStatus.IterationLimitExceeded
    assert 0.1 < res.snapshot.volume_fraction < 0.5
    assert res.snapshot.iteration_count == 5
    assert violations(res.snapshot, 1e-12) == 0


def test_progress_sees_every_iteration():
    snap = disk_start(50, 0.1, 13)
    seen = []
    res = srm.srm_generate(snap, srm.SrmParams(c_w=0.05, c_m=0.01, f_target=0.3), progress=seen.append)
    assert [r.iteration for r in seen] == list(range(1, len(seen) + 1))
    assert len(seen) == res.snapshot.iteration_count
    assert seen[-1].volume_fraction == pytest.approx(res.snapshot.volume_fraction)


def test_parameter_validation():
    snap = disk_start(10, 0.1, 2)
    for kw in (dict(c_w=-0.01), dict(c_w=0.26), dict(f_target=0.0), dict(f_target=1.0), dict(n_k=0),
               dict(c_w=0.0, f_target=0.9), dict(c_m=0.5)):
        with pytest.raises(srm.ValidationError):
            srm.srm_generate(snap, srm.SrmParams(**kw))
    srm.srm_generate(snap, srm.SrmParams(c_w=0.25, f_target=0.12))
    with pytest.raises(srm.ValidationError):
        srm.srm_generate(srm.Snapshot([1.0, 1.0], np.zeros((0, 2)), np.zeros(0)), srm.SrmParams())


def test_relax_zero_step_identity_and_validity():
    snap = disk_start(100, 0.2, 5)
    before = snap.copy()
    srm.relax_sweeps(snap, 0.0, 0.0, 4, 3, 1)
    assert np.array_equal(snap.pos, before.pos)
    snap = disk_start(200, 0.3, 21)
    srm.relax_sweeps(snap, 0.01, 0.0, 8, 5, 2)
    assert violations(snap, 0.0) == 0
    snap = disk_start(150, 0.45, 8)
    srm.shake(snap, srm.SrmParams(c_m=0.005, n_k=6, n_l=8), 4)
    assert violations(snap, 0.0) == 0


def test_swell_all():
    snap = disk_start(50, 0.1, 3)
    before = snap.copy()
    srm.swell_all(snap, 0.02)
    assert np.array_equal(snap.pos, before.pos)
    assert np.array_equal(snap.radius, before.radius * 1.02)
    s0 = snap.copy()
    srm.swell_all(s0, 0.0)
    assert np.array_equal(s0.radius, snap.radius)
