"""Golden vectors for the offline preprocessing kernels, from the reference.

TEST INFRASTRUCTURE. Runs only in the build container (needs oracle/_ref: the reference trijoin
built from /root/reference/proj by oracle/Makefile). Every expected value is an output of the
reference's own code, through oracle/ref_shim.cpp:
  * ladders: build_lod_ladder (proj/src/simplify.cpp; hd / ph of every coarse level,
    :229-251; hd = compute_facet_hd, proj/src/hausdorff.cpp:15-27) of reference-generated
    meshes (sphere, tube, torus, a radially noisy sphere) at lods [20, 60, 100], hd_grid 8;
  * hd_direct: compute_facet_hd of off-surface query triangles at grids 1, 3 and 8;
  * voxelize: proj/src/voxelize.cpp:27-79 on each coarsest level for several k and seeds.

    python tests/golden/make_preprocess.py
"""
import ctypes
import os
import struct
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
import trijoin as ref  # noqa: E402

shim = ctypes.CDLL(os.path.join(ROOT, "oracle", "_ref", "libref_shim.so"))
shim.ref_last_error.restype = ctypes.c_char_p
DP = ctypes.POINTER(ctypes.c_double)
UP = ctypes.POINTER(ctypes.c_uint32)
IP = ctypes.POINTER(ctypes.c_int32)


def gen_mesh(shape, facets, scale, seed):
    with tempfile.TemporaryDirectory() as d:
        ref.generate(d, shape=shape, facets=facets, scale=scale, count=1, seed=seed)
        off = [f for f in sorted(os.listdir(d)) if f.endswith(".off")][0]
        v, f = ref.parse_off(open(os.path.join(d, off)).read())
    return np.asarray(v, dtype=np.float64).reshape(-1, 3), np.asarray(f, dtype=np.uint32).reshape(-1, 3)


def ladder(v, f, lods, grid):
    lods = np.asarray(lods, dtype=np.int32)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "ladder.bin")
        rc = shim.ref_build_ladder(np.ascontiguousarray(v).ctypes.data_as(DP), ctypes.c_uint64(len(v)),
                                   np.ascontiguousarray(f).ctypes.data_as(UP), ctypes.c_uint64(len(f)),
                                   lods.ctypes.data_as(IP), ctypes.c_uint32(len(lods)), ctypes.c_int32(grid),
                                   path.encode())
        assert rc == 0, shim.ref_last_error()
        b = open(path, "rb").read()
    o = 0

    def rd(fmt):
        nonlocal o
        r = struct.unpack_from(fmt, b, o)
        o += struct.calcsize(fmt)
        return r

    levels = []
    (nl,) = rd("<I")
    for _ in range(nl):
        lv, cl, nv, nf = rd("<iBQQ")
        verts = np.frombuffer(b, np.float64, 3 * nv, o).reshape(nv, 3); o += 24 * nv
        fac = np.frombuffer(b, np.uint32, 3 * nf, o).reshape(nf, 3); o += 12 * nf
        (nh,) = rd("<Q"); hd = np.frombuffer(b, np.float64, nh, o); o += 8 * nh
        (npd,) = rd("<Q"); ph = np.frombuffer(b, np.float64, npd, o); o += 8 * npd
        (na,) = rd("<Q"); anc = np.frombuffer(b, np.uint32, na, o); o += 4 * na
        levels.append(dict(level=lv, verts=verts.copy(), facets=fac.copy(), hd=hd.copy(), ph=ph.copy(), anc=anc.copy()))
    return levels


def facet_hd(v, f, tris, grid):
    out = np.zeros(len(tris))
    rc = shim.ref_facet_hd(np.ascontiguousarray(v).ctypes.data_as(DP), ctypes.c_uint64(len(v)),
                           np.ascontiguousarray(f).ctypes.data_as(UP), ctypes.c_uint64(len(f)), ctypes.c_uint64(len(tris)),
                           np.ascontiguousarray(tris).ctypes.data_as(DP), ctypes.c_int32(grid), out.ctypes.data_as(DP))
    assert rc == 0, shim.ref_last_error()
    return out


def voxelize(v, f, k, seed):
    out = np.zeros(len(f), dtype=np.uint32)
    rc = shim.ref_voxelize(np.ascontiguousarray(v).ctypes.data_as(DP), ctypes.c_uint64(len(v)),
                           np.ascontiguousarray(f).ctypes.data_as(UP), ctypes.c_uint64(len(f)), ctypes.c_uint32(k),
                           ctypes.c_uint64(seed), out.ctypes.data_as(UP))
    assert rc == 0, shim.ref_last_error()
    return out


def main():
    rng = np.random.default_rng(20261018)
    meshes = [("sphere", 300, 0.35, 21), ("tube", 1000, 3.0, 31), ("torus", 600, 1.5, 7), ("sphere", 2000, 2.0, 5)]
    out = {}
    for mi, (shape, nfac, scale, seed) in enumerate(meshes):
        v, f = gen_mesh(shape, nfac, scale, seed)
        if mi == 3:  # radially noisy "scanned" sphere, translated away from the origin
            r = np.linalg.norm(v, axis=1, keepdims=True)
            v = v * (1.0 + 0.05 * rng.standard_normal((len(v), 1))) + np.array([40.0, -7.5, 12.25])
            del r
        out[f"m{mi}_verts"], out[f"m{mi}_facets"] = v, f
        lv = ladder(v, f, [20, 60, 100], 8)
        for li, L in enumerate(lv):
            for key in ("verts", "facets", "hd", "ph", "anc"):
                out[f"m{mi}_l{li}_{key}"] = L[key]
            out[f"m{mi}_l{li}_level"] = np.int32(L["level"])
        # direct compute_facet_hd on perturbed copies of the original facets (off the surface)
        sel = rng.choice(len(f), size=min(200, len(f)), replace=False)
        tris = v[f[sel]].reshape(-1, 9) + rng.normal(0, 0.02 * scale, (len(sel), 9))
        out[f"m{mi}_qtris"] = tris
        for g in (1, 3, 8):
            out[f"m{mi}_qhd_g{g}"] = facet_hd(v, f, tris, g)
        # voxelize on the coarsest level
        c = lv[0]
        for k, s in ((1, 3), (5, 11), (int(np.ceil(0.02 * len(f))), 0x9E3779B97F4A7C15 * (mi + 1) % (1 << 64)),
                     (37, 12345), (len(c["facets"]) + 3, 99)):
            out[f"m{mi}_vox_k{k}_s{s}"] = voxelize(c["verts"], c["facets"], k, s)
    out["n_meshes"] = np.int32(len(meshes))
    # the C++ drop-in test (tests/cpp/test_preprocess.cpp) reads mesh 1 in a raw little-endian form:
    #   u64 nv, nf; f64 verts[3 nv]; u32 facets[3 nf]; u32 n_levels; per level: i32 level,
    #   u64 lnv, lnf, f64 verts, u32 facets, f64 hd[lnf], f64 ph[lnf], u32 anc[nf];
    #   u32 k, u64 seed, u32 labels[coarsest lnf]
    m = 1
    key = [k for k in out if k.startswith(f"m{m}_vox_k37_")][0]
    with open(os.path.join(HERE, "preprocess_m1.bin"), "wb") as fp:
        v, f = out[f"m{m}_verts"], out[f"m{m}_facets"]
        fp.write(struct.pack("<QQ", len(v), len(f)) + v.astype("<f8").tobytes() + f.astype("<u4").tobytes())
        fp.write(struct.pack("<I", 3))
        for li in range(3):
            lv, lf = out[f"m{m}_l{li}_verts"], out[f"m{m}_l{li}_facets"]
            fp.write(struct.pack("<iQQ", int(out[f"m{m}_l{li}_level"]), len(lv), len(lf)))
            fp.write(lv.astype("<f8").tobytes() + lf.astype("<u4").tobytes())
            fp.write(out[f"m{m}_l{li}_hd"].astype("<f8").tobytes() + out[f"m{m}_l{li}_ph"].astype("<f8").tobytes())
            fp.write(out[f"m{m}_l{li}_anc"].astype("<u4").tobytes())
        fp.write(struct.pack("<IQ", 37, 12345) + out[key].astype("<u4").tobytes())
    np.savez_compressed(os.path.join(HERE, "preprocess.npz"), **out)
    print("wrote", os.path.join(HERE, "preprocess.npz"), sum(a.nbytes for a in out.values()), "bytes")


if __name__ == "__main__":
    main()
