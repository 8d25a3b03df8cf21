"""API-level behaviour of the device path that the reference's engine contract implies:
live progress during the device-resident generate loop (engine.hpp:251-254: the sink
sees every iteration, as it ends), the cached generate graph, and the argument checks of
the AoS record upload (geometry.hpp:139-144 layout)."""
import ctypes as C
import time

import numpy as np
import pytest

import orc
import paper_2605_18254_b200 as srm
from paper_2605_18254_b200 import _native

pytestmark = pytest.mark.gpu


def _disks(n, f0, seed):
    r = np.sqrt(f0 / (n * np.pi))
    pos, ids = srm.rsa_place(np.full(n, r), [1.0, 1.0], srm.K_RSA_DEFAULT_ATTEMPTS, seed)
    return pos, np.full(n, r), ids


def test_progress_is_live_and_complete_beyond_the_ring():
    """> 4096 iterations (the mapped ring's size): every record arrives, in order, and the
    first ones arrive while the graph is still running."""
    pos, r, ids = _disks(64, 0.1, 3)
    seen, t_seen = [], []
    with srm.Context([1.0, 1.0], 64) as ctx:
        ctx.upload(pos, r, ids)
        p = srm.SrmParams(c_w=5e-5, c_m=0.002, n_k=2, n_l=4, f_target=0.2, seed=9)
        t0 = time.perf_counter()
        out = ctx.generate(p, 0, lambda rec: (seen.append(rec), t_seen.append(time.perf_counter())))
        t1 = time.perf_counter()
    assert out.status == srm.OK
    assert out.iteration_count > 4096
    assert [s.iteration for s in seen] == list(range(1, out.iteration_count + 1))
    assert all(a.elapsed_seconds <= b.elapsed_seconds for a, b in zip(seen, seen[1:]))
    assert seen[-1].volume_fraction == pytest.approx(0.2, rel=1e-12)
    # delivered during the run, not after it: the first record long before the return
    assert t_seen[0] - t0 < 0.5 * (t1 - t0)


def test_progress_sink_exception_propagates_after_the_run():
    pos, r, ids = _disks(50, 0.1, 4)
    calls = []

    def sink(rec):
        calls.append(rec.iteration)
        if rec.iteration == 3:
            raise RuntimeError("stop")

    snap = srm.Snapshot([1.0, 1.0], pos, r, ids)
    # the python sink runs inside a ctypes callback: its exception is reported, the run
    # itself completes and stays usable
    res = srm.srm_generate(snap, srm.SrmParams(c_w=0.05, c_m=0.01, f_target=0.3, seed=2), progress=sink)
    assert res.status == srm.GenerateStatus.Converged
    assert calls[:3] == [1, 2, 3]


def test_generate_graph_is_cached_between_calls():
    pos, r, ids = _disks(200, 0.1, 5)
    p = srm.SrmParams(c_w=0.05, c_m=0.005, n_k=6, n_l=6, f_target=0.4, seed=11)
    with srm.Context([1.0, 1.0], 200) as ctx:
        ctx.upload(pos, r, ids)
        a = ctx.generate(p)
        xa, ra, ia = ctx.download()
        ctx.upload(pos, r, ids)
        b = ctx.generate(p)
        xb, rb, ib = ctx.download()
        builds = ctx.graph_builds()
    assert builds == 1
    assert a.iteration_count == b.iteration_count and a.rounds == b.rounds
    assert np.array_equal(xa, xb) and np.array_equal(ra, rb) and np.array_equal(ia, ib)
    with srm.Context([1.0, 1.0], 200) as fresh:  # same as a fresh context
        fresh.upload(pos, r, ids)
        fresh.generate(p)
        xc, _, _ = fresh.download()
    assert np.array_equal(xa, xc)


def _records(n, dtype):
    rec = np.zeros(n, dtype)
    pos, r = orc.random_particles(n, 3, 0.001, 0.002, [1.0] * 3, 2)
    rec["id"] = np.arange(n)
    rec["pos"] = pos
    rec["radius"] = r
    return rec


def test_upload_records_rejects_bad_layouts():
    lib = _native.lib()
    packed = np.dtype([("id", "<i4"), ("pos", "<f8", 3), ("radius", "<f8")])  # off_pos = 4
    rec = _records(100, packed)
    with srm.Context([1.0] * 3, 100) as ctx:
        with pytest.raises(srm.ValidationError):
            ctx.upload_records(rec, 0, 4, 28)  # the Python check: unaligned dtype
        ptr = rec.ctypes.data_as(C.c_void_p)
        # the C ABI itself: misaligned offsets, fields outside the stride, null records
        assert lib.srm_b200_upload_records(ctx.handle, 100, ptr, 36, 0, 4, 28) == srm.INVALID
        assert lib.srm_b200_upload_records(ctx.handle, 100, ptr, 40, 0, 8, 40) == srm.INVALID
        assert lib.srm_b200_upload_records(ctx.handle, 100, None, 40, 0, 8, 32) == srm.INVALID
        assert lib.srm_b200_upload_records(ctx.handle, 100, ptr, 40, 38, 8, 32) == srm.INVALID
        ctx.sync()  # the context is still healthy: no sticky CUDA error
    with srm.Context([1.0] * 3, 100, shape="platelet") as pctx:
        aligned = np.dtype({"names": ["id", "pos", "radius"], "formats": ["<i4", ("<f8", 3), "<f8"],
                            "offsets": [0, 8, 32], "itemsize": 40})
        ok = _records(100, aligned)
        assert lib.srm_b200_upload_records(pctx.handle, 100, ok.ctypes.data_as(C.c_void_p), 40, 0, 8,
                                           32) == srm.INVALID
