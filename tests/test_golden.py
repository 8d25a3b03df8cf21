"""The oracle and the product's host code against the committed golden fixtures
(tests/golden/*.npz, generated from the reference by tests/golden/make_golden.py).
Runs without /root/reference."""
import os

import numpy as np
import pytest

import orc
import paper_2605_18254_b200 as srm

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(G, name + ".npz"))


@pytest.mark.parametrize("name", ["grid_2d", "grid_3d"])
def test_oracle_keys_order_collisions_vs_golden(name):
    z = load(name)
    pos, r, L, cs = z["pos"], z["r"], list(z["L"]), float(z["cs"])
    dim = pos.shape[1]
    keys, dims, _ = orc.o_keys(dim, L, cs, pos)
    assert np.array_equal(keys.astype(np.uint64), z["keys"])
    order, _ = orc.o_sort(keys, np.arange(len(r), dtype=np.int32), int(np.prod(dims)))
    assert np.array_equal(z["remap"][order], np.arange(len(r)))
    st = orc.o_stats(dim, L, pos, r)
    assert (st.overlap_pairs > 0) == bool(z["any"])
    # per-particle collision flags: particle i overlaps some j
    hit = np.zeros(len(r), bool)
    for i in range(len(r)):
        d = pos - pos[i]
        d -= np.asarray(L) * np.rint(d / np.asarray(L))
        rr = r + r[i]
        m = (d * d).sum(1) <= rr * rr
        m[i] = False
        hit[i] = m.any()
    assert np.array_equal(hit, z["per"].astype(bool))


@pytest.mark.parametrize("name", ["rsa_2d", "rsa_3d"])
def test_product_rsa_vs_golden(name):
    z = load(name)
    n = len(z["ids"])
    pos, ids = srm.rsa_place(np.full(n, float(z["r"])), list(z["L"]), srm.K_RSA_DEFAULT_ATTEMPTS, int(z["seed"]))
    assert np.array_equal(pos, z["pos"]) and np.array_equal(ids, z["ids"])


@pytest.mark.parametrize("name", ["e2e_2d", "e2e_3d"])
def test_reference_e2e_fixture_sane(name):
    z = load(name)
    assert np.all(np.abs(z["f"] / z["f_t"] - 1.0) < 1e-9)
    assert z["nnd"].shape == (len(z["seeds"]), int(z["n"]))
    assert np.all(z["nnd"] >= 2.0 * z["r_target"] * (1 - 1e-9))  # no overlaps
