"""Offline preprocessing on the GPU through the C-ABI, bitwise against the
reference's own outputs (tests/golden/preprocess.npz, made by tests/golden/make_preprocess.py
from proj/src/simplify.cpp build_lod_ladder, hausdorff.cpp compute_facet_hd and voxelize.cpp)."""
import re

import numpy as np
import pytest

import tjtest
from tjtest import bits, golden

pytestmark = pytest.mark.gpu

G = np.load(golden("preprocess.npz"))
N_MESHES = int(G["n_meshes"])


def mesh(m):
    return G[f"m{m}_verts"], G[f"m{m}_facets"]


def level(m, li):
    return G[f"m{m}_l{li}_verts"], G[f"m{m}_l{li}_facets"]


def tris(v, f):
    return np.asarray(v)[np.asarray(f)].reshape(-1, 9)


@pytest.mark.parametrize("m", range(N_MESHES))
def test_ladder_hd_bitexact(capi, m):
    """hd of every facet of the coarse levels (src/simplify.cpp:233-234, hausdorff.cpp:15-27)."""
    for li in (0, 1):
        out = capi.facet_hd([mesh(m)], [tris(*level(m, li))], 8)
        assert (bits(out) == bits(G[f"m{m}_l{li}_hd"])).all(), (m, li)


def test_ladder_hd_all_meshes_one_batch(capi):
    """Every (mesh, level) in one batched call gives the same bits as the reference."""
    ms, qs, want = [], [], []
    for m in range(N_MESHES):
        for li in (0, 1):
            ms.append(mesh(m))
            qs.append(tris(*level(m, li)))
            want.append(G[f"m{m}_l{li}_hd"])
    out = capi.facet_hd(ms, qs, 8)
    assert (bits(out) == bits(np.concatenate(want))).all()


@pytest.mark.parametrize("m", range(N_MESHES))
@pytest.mark.parametrize("grid", [1, 3, 8])
def test_facet_hd_direct_bitexact(capi, m, grid):
    """compute_facet_hd of off-surface triangles (perturbed original facets) at several grids."""
    out = capi.facet_hd([mesh(m)], [G[f"m{m}_qtris"]], grid)
    assert (bits(out) == bits(G[f"m{m}_qhd_g{grid}"])).all()


@pytest.mark.parametrize("m", range(N_MESHES))
def test_ladder_ph_bitexact(capi, m):
    """ph of every facet of the coarse levels (src/simplify.cpp:238-251)."""
    for li in (0, 1):
        out = capi.facet_ph([mesh(m)], [tris(*level(m, li))], [G[f"m{m}_l{li}_anc"]])
        assert (bits(out) == bits(G[f"m{m}_l{li}_ph"])).all(), (m, li)


def test_level100_paddings_zero_in_golden():
    """include/trijoin/mesh.hpp:57: hd / ph are identically 0 at level 100 (what the batched C++
    fill writes without a GPU pass)."""
    for m in range(N_MESHES):
        assert not G[f"m{m}_l2_hd"].any() and not G[f"m{m}_l2_ph"].any()


def test_voxelize_bitexact(capi):
    """voxelize (src/voxelize.cpp:27-79) on each coarsest level for several (k, seed), all in
    one batched call; k above the facet count and k = 1 included."""
    ms, ks, ss, want = [], [], [], []
    for key in G.files:
        mm = re.fullmatch(r"m(\d+)_vox_k(\d+)_s(\d+)", key)
        if not mm:
            continue
        m, k, s = int(mm.group(1)), int(mm.group(2)), int(mm.group(3))
        ms.append(level(m, 0))
        ks.append(k)
        ss.append(s)
        want.append(G[key])
    assert len(ms) >= 16
    out = capi.voxelize(ms, ks, ss)
    for o, w, k in zip(out, want, ks):
        assert (o == w).all(), k


def test_preprocess_rejects_bad_input(capi):
    v, f = mesh(0)
    bad = f.copy()
    bad[0, 0] = len(v)  # vertex id out of range
    with pytest.raises(RuntimeError, match="status 1"):
        capi.facet_hd([(v, bad)], [tris(v, f)[:2]], 8)
    with pytest.raises(RuntimeError, match="status 1"):
        capi.facet_hd([(v, f)], [tris(v, f)[:2]], 0)
    with pytest.raises(RuntimeError, match="status 1"):
        capi.voxelize([(v, f)], [0], [1])
    anc = np.zeros(len(f), np.uint32)
    anc[3] = 5  # ancestor beyond the one-facet LOD
    with pytest.raises(RuntimeError, match="status 1"):
        capi.facet_ph([(v, f)], [tris(v, f)[:1]], [anc])


def test_cpp_dropin_preprocess_api():
    """The C++ drop-in (trijoin::fill_ladder_paddings, compute_facet_hd / _ph,
    hd_covering_radius, voxelize) bitwise against the reference on one mesh
    (tests/cpp/test_preprocess.cpp)."""
    import os
    import subprocess
    exe = os.path.join(tjtest.ROOT, "tests", "cpp", "test_preprocess")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(tjtest.ROOT, "tests", "cpp"), "test_preprocess"], check=True)
    p = subprocess.run([exe, golden("preprocess_m1.bin")], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failed" in p.stdout
