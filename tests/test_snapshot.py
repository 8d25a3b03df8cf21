"""The snapshot codec: srm_b200_snapshot_encode writes the
reference's own SRMSNAP file bytes -- binary (snapshot_io.cpp:170-191) and text
(snapshot_io.cpp:150-167) -- byte for byte against the reference's snapshot_to_binary /
snapshot_to_text (oracle/_ref, built from snapshot_io.cpp), for disks, spheres and
platelets, with awkward doubles in the header and rows; and the files round-trip through
snapshot_info.  CPU only (the device save/load is in tests/test_gpu_snapshot.py)."""
import ctypes as C
import os

import numpy as np
import pytest

import orc
import paper_2605_18254_b200 as srm


def ref_bytes(dim, shape, L, pos, r, nrm, D, t, ids, f, it, seed, p, binary):
    lib = orc.ref()
    fn = lib.ref_snapshot_bytes
    fn.restype = C.c_int64
    vp = C.c_void_p
    fn.argtypes = [C.c_int, C.c_int, vp, C.c_int64, vp, vp, vp, vp, vp, vp, C.c_double, C.c_int64, C.c_uint64, vp,
                   vp, C.c_int, vp, C.c_int64]
    pd = np.array([p.c_w, p.c_m, p.c_r, p.f_target])
    pi = np.array([p.n_k, p.n_l, p.max_iterations, p.seed, p.reorder_period], np.uint64).view(np.int64)
    Lp = np.asarray(L, np.float64)

    def P(a):
        return None if a is None else np.ascontiguousarray(a).ctypes.data_as(vp)
    args = [dim, shape, P(Lp), len(ids), P(pos), P(r), P(nrm), P(D), P(t), P(ids), f, it, seed, P(pd), P(pi),
            1 if binary else 0]
    n = fn(*args, None, 0)
    buf = C.create_string_buffer(int(n))
    fn(*args, buf, n)
    return buf.raw[:n]


def _params():
    return srm.SrmParams(c_w=0.02, c_m=1.0 / 3.0, c_r=0.012, n_k=10, n_l=20, f_target=0.3, max_iterations=123456,
                         seed=(1 << 63) + 12345, reorder_period=16)


@pytest.mark.parametrize("binary", [True, False])
@pytest.mark.parametrize("dim", [2, 3])
def test_sphere_snapshot_bytes_match_reference(dim, binary):
    rng = np.random.default_rng(dim + 7 * binary)
    n = 257
    L = [1.0, 0.7, 1.3][:dim]
    pos = rng.uniform(0, 1, (n, dim)) * L
    pos[0] = 0.0
    pos[1, 0] = 1e-300
    r = rng.uniform(1e-3, 2e-3, n)
    r[2] = 1.0 / 3.0
    ids = rng.permutation(n).astype(np.int32)
    f, it, seed, p = 0.123456789012345678, 42, 2 ** 64 - 1, _params()
    mine = srm.snapshot_bytes(L, pos, r, ids, volume_fraction=f, iteration_count=it, seed=seed, params=p,
                              binary=binary)
    ref = ref_bytes(dim, 0, L, pos, r, None, None, None, ids, f, it, seed, p, binary)
    assert mine == ref


@pytest.mark.parametrize("binary", [True, False])
def test_platelet_snapshot_bytes_match_reference(binary):
    rng = np.random.default_rng(5)
    n = 100
    L = [25.01, 25.01, 25.01]
    pos = rng.uniform(0, 25.01, (n, 3))
    nrm = rng.normal(size=(n, 3))
    nrm /= np.linalg.norm(nrm, axis=1)[:, None]
    D = np.full(n, 0.8183)
    t = D / 100.0
    ids = np.arange(n, dtype=np.int32)
    p = _params()
    mine = srm.snapshot_bytes(L, pos, None, ids, normal=nrm, diameter=D, thickness=t, volume_fraction=0.05,
                              iteration_count=7, seed=3, params=p, binary=binary)
    ref = ref_bytes(3, 1, L, pos, None, nrm, D, t, ids, 0.05, 7, 3, p, binary)
    assert mine == ref


def test_snapshot_info_reads_reference_files(tmp_path):
    rng = np.random.default_rng(1)
    pos = rng.uniform(0, 1, (50, 3))
    r = np.full(50, 0.01)
    p = _params()
    for binary in (True, False):
        path = os.path.join(tmp_path, f"s{int(binary)}.srm")
        with open(path, "wb") as fh:
            fh.write(ref_bytes(3, 0, [1.0, 1.0, 1.0], pos, r, None, None, None, np.arange(50, dtype=np.int32),
                               0.25, 9, 11, p, binary))
        info = srm.snapshot_info(path)
        assert info["dim"] == 3 and info["shape"] == "sphere" and info["count"] == 50
        assert info["box"] == [1.0, 1.0, 1.0] and info["volume_fraction"] == 0.25
        assert info["iteration_count"] == 9 and info["seed"] == 11
        assert info["params"].c_m == p.c_m and info["params"].seed == p.seed
    bad = os.path.join(tmp_path, "bad.srm")
    with open(bad, "wb") as fh:
        fh.write(b"SRMSNAP\0\x02\0\0\0")
    with pytest.raises(srm.IoError):
        srm.snapshot_info(bad)
