"""Device checkpoint / resume through the reference's snapshot format (SURVEY.md §8f
row 4): a context's state saved with srm_b200_save_snapshot (binary and text) equals
the host encoder's bytes (itself byte-identical to the reference's: tests/test_snapshot.py)
and loads back into a fresh context bit for bit; spheres and platelets; a generate run
resumed from a checkpoint reaches the target with zero overlaps."""
import os

import numpy as np
import pytest

import orc
import paper_2605_18254_b200 as srm

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("binary", [True, False])
def test_sphere_roundtrip(tmp_path, binary):
    n, L = 3000, [1.0, 1.0, 1.0]
    r0 = (0.2 / (n * 4.0 / 3.0 * np.pi)) ** (1.0 / 3.0)
    pos, ids = srm.rsa_place(np.full(n, r0), L, 10000, 3)
    p = srm.SrmParams(c_w=0.02, c_m=0.1 * r0, n_k=10, n_l=10, f_target=0.3, seed=5)
    path = os.path.join(tmp_path, "s.srm")
    with srm.Context(L, n) as ctx:
        ctx.upload(pos, np.full(n, r0), ids)
        out = ctx.generate(srm.SrmParams(c_w=0.02, c_m=0.1 * r0, n_k=10, n_l=10, f_target=0.25, seed=5))
        ctx.save_snapshot(path, out.volume_fraction, out.iteration_count, 5, p, binary=binary)
        a = ctx.download()
    with open(path, "rb") as fh:
        data = fh.read()
    assert data == srm.snapshot_bytes(L, a[0], a[1], a[2], volume_fraction=out.volume_fraction,
                                      iteration_count=out.iteration_count, seed=5, params=p, binary=binary)
    info = srm.snapshot_info(path)
    assert info["count"] == n and info["iteration_count"] == out.iteration_count
    with srm.Context(L, n) as ctx:
        ctx.load_snapshot(path)
        b = ctx.download()
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
        res = ctx.generate(p, iteration_count=info["iteration_count"])
        assert abs(res.volume_fraction / 0.3 - 1.0) < 1e-9
        pos2, r2, _ = ctx.download()
    assert orc.o_stats(3, L, pos2, r2).overlap_pairs == 0


def test_platelet_roundtrip(tmp_path):
    L = [6.0, 6.0, 6.0]
    pos, nrm, ids = srm.rsa_platelets(300, 1.0, 20.0, L, 10000, 4)
    D = np.full(300, 1.0)
    path = os.path.join(tmp_path, "p.srm")
    with srm.Context(L, 300, shape="platelet") as ctx:
        ctx.upload_platelets(pos, nrm, D, D / 20.0, ids)
        ctx.save_snapshot(path, 0.01, 0, 4)
        a = ctx.download_platelets()
    with srm.Context(L, 300, shape="platelet") as ctx:
        ctx.load_snapshot(path)
        b = ctx.download_platelets()
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    with srm.Context([5.0, 5.0, 5.0], 300, shape="platelet") as ctx:
        with pytest.raises(srm.ValidationError):
            ctx.load_snapshot(path)  # another box
