"""Host-side pieces of the product that run without a GPU:

* rsa_place (libsrm_b200.so host code) is bit-identical to the reference's rsa_place
  (rsa.hpp:21-61) for the same seed, including its failure modes (test_rsa.cpp);
* mix_seed equals random.hpp:84-89;
* the C-ABI library loads and exports every symbol include/srm_b200.h declares;
* without a device the product refuses to run (no CPU fallback).
"""
import os
import re

import numpy as np
import pytest

import orc
import paper_2605_18254_b200 as srm
from paper_2605_18254_b200 import _native

ROOT = orc.ROOT


@pytest.mark.parametrize("dim,n,f,seed,L", [
    (2, 1000, 0.1, 42, [1.0, 1.0]),
    (3, 200, None, 5, [1.0, 1.0, 1.0]),
    (3, 5000, 0.25, 7, [1.0, 1.0, 1.0]),
    (2, 3000, 0.4, 9, [2.0, 1.0]),
    (3, 2000, 0.2, 13, [1.0, 1.3, 0.7]),
])
def test_rsa_bit_identical_to_reference(dim, n, f, seed, L):
    unit = np.pi if dim == 2 else 4.0 / 3.0 * np.pi
    r = 0.03 if f is None else (f * np.prod(L) / (n * unit)) ** (1.0 / dim)
    radii = np.full(n, r)
    st, pos_r, ids_r, _ = orc.r_rsa(dim, L, radii, 10000, seed)
    assert st == 0
    pos, ids = srm.rsa_place(radii, L, 10000, seed)
    assert np.array_equal(pos, pos_r)
    assert np.array_equal(ids, ids_r)


def test_rsa_polydisperse_bit_identical():
    rng = np.random.default_rng(3)
    radii = np.clip(rng.lognormal(-0.0196, 0.198, 3000), 0.5, 2.0) * 0.004
    L = [1.0, 1.0, 1.0]
    st, pos_r, _, _ = orc.r_rsa(3, L, radii, 10000, 77)
    assert st == 0
    pos, _ = srm.rsa_place(radii, L, 10000, 77)
    assert np.array_equal(pos, pos_r)


def test_rsa_failure_and_validation():
    # test_rsa.cpp:70-91
    with pytest.raises(srm.PlacementFailure) as e:
        srm.rsa_place(np.full(10, 0.24), [1.0, 1.0], 50, 2)
    st, _, _, placed = orc.r_rsa(2, [1.0, 1.0], np.full(10, 0.24), 50, 2)
    assert st == 2 and e.value.placed_count == placed < 10 and e.value.attempt_limit == 50
    for bad in ([], [0.0], [-0.1], [0.25]):
        with pytest.raises(srm.ValidationError):
            srm.rsa_place(np.asarray(bad, float), [1.0, 1.0], 10, 1)
    pos, ids = srm.rsa_place([0.249], [1.0, 1.0], 10, 1)
    assert pos.shape == (1, 2) and ids[0] == 0
    pos, ids = srm.rsa_place([0.2], [1.0, 1.0], 1, 1)  # one attempt suffices
    assert 0.0 <= pos[0, 0] < 1.0 and 0.0 <= pos[0, 1] < 1.0


def test_mix_seed_matches_reference():
    for s, t in [(1, 0), (42, 10000), (2**63 + 5, 7), (0, 2**40)]:
        assert srm.mix_seed(s, t) == orc.ref().ref_mix_seed(s, t)


def test_abi_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "srm_b200.h")).read()
    declared = set(re.findall(r"\b(srm_b200_[a-z0-9_]+)\s*\(", header))
    declared = {d for d in declared if d not in ("srm_b200_progress_fn",)}
    lib = _native.lib()
    missing = [d for d in sorted(declared) if not hasattr(lib, d)]
    assert not missing, missing
    assert declared <= set(_native.EXPORTED) | {"srm_b200_progress_fn"}


def test_header_compiles_as_c():
    import subprocess
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "t.c")
        with open(src, "w") as fh:
            fh.write('#include "srm_b200.h"\nint main(void){srm_b200_params p; (void)p; return 0;}\n')
        r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                            "-c", src, "-o", os.path.join(d, "t.o")], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


def test_no_device_fails_loudly():
    import conftest
    if conftest._has_gpu():
        pytest.skip("a GPU is present")
    with pytest.raises(srm.NoDeviceError):
        srm.Context([1.0, 1.0], 10)


def test_create_rejects_capacity_beyond_int32():
    # sorted indices and near-list entries are int32: refused before any
    # device work, so this holds with or without a GPU
    with pytest.raises(srm.ValidationError):
        srm.Context([1.0, 1.0, 1.0], 2**31)
