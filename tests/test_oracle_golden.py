"""The C restatement oracle (oracle/tj_oracle.c) pinned against the reference's golden vectors
(tests/golden/, produced by the reference itself). CPU only."""
import numpy as np
import pytest

import tjtest
from tjtest import PD, PU32, PU64, bits, golden, ptr


@pytest.mark.parametrize("name", ["tritri_seed42.npz", "tritri_seed20240817.npz", "tritri_analytic.npz"])
def test_oracle_tri_tri_bitexact(oracle_lib, name):
    g = np.load(golden(name))
    out = np.zeros(len(g["d"]))
    oracle_lib.ora_tri_tri_batch(np.uint64(len(out)).item(), ptr(np.ascontiguousarray(g["a"])),
                                 ptr(np.ascontiguousarray(g["b"])), ptr(out))
    assert (bits(out) == bits(g["d"])).all()


def test_oracle_analytic_values(oracle_lib):
    g = np.load(golden("tritri_analytic.npz"))
    np.testing.assert_allclose(g["d"], g["expect"], atol=1e-12)  # proj/tests/acceptance.cpp:514-533


def test_oracle_mindist_bitexact(oracle_lib):
    g = np.load(golden("mindist_random.npz"))
    out = np.zeros(len(g["d"]))
    oracle_lib.ora_mindist_batch(np.uint64(len(out)).item(), ptr(np.ascontiguousarray(g["a"])),
                                 ptr(np.ascontiguousarray(g["b"])), ptr(out))
    assert (bits(out) == bits(g["d"])).all()


@pytest.mark.parametrize("j", tjtest.golden_joins() + tjtest.adversarial_joins(), ids=tjtest.join_id)
def test_oracle_join_matches_reference(oracle_lib, j):
    kw = dict(j["kwargs"])
    lods = kw.pop("lods", [20, 40, 60, 80, 100])
    s = golden(j["s"] + ".idx") if j["s"] else ""
    recs, stages = tjtest.oracle_join(oracle_lib, golden(j["r"] + ".idx"), s, lods=lods, **kw)
    assert recs == j["records"]
    assert stages == j["stages"]
