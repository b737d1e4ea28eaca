"""Regenerate the golden fixtures of tests/golden/ from the reference itself.

TEST INFRASTRUCTURE. Runs only in the build container (needs oracle/_ref, i.e. the reference
trijoin built from /root/reference/proj by oracle/Makefile). Every expected value here is
an output of the reference's own code:
  * tri-tri / mindist vectors: proj/src/geom.cpp through oracle/ref_shim.cpp, on the inputs
    of the reference tests (proj/tests/test_geom.cpp:95-110 seed 42, 2000 pairs;
    proj/tests/acceptance.cpp:499-512 seed 20240817, 10000 pairs; the analytic cases of
    proj/tests/test_geom.cpp:70-93);
  * datasets: proj/tests/helpers.hpp mini_dataset(...) and the reference generator /
    preprocessor (trijoin.generate / trijoin.preprocess);
  * joins: the reference trijoin.join records and stage statistics (minus wall times);
  * staged refine bounds: proj/tests/test_refine.cpp:21-39-style staging, then the
    reference gather_facet_data + refine_kernel per level (ref_staged_dump).

    python tests/golden/make_golden.py
"""
import ctypes
import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
import trijoin as ref  # noqa: E402

P = ctypes.POINTER(ctypes.c_double)
shim = ctypes.CDLL(os.path.join(ROOT, "oracle", "_ref", "libref_shim.so"))
shim.ref_last_error.restype = ctypes.c_char_p


def tri_pairs(seed, n, lo, hi, size):
    a = np.zeros((n, 9))
    b = np.zeros((n, 9))
    d = np.zeros(n)
    shim.ref_random_tri_pairs(ctypes.c_uint64(seed), ctypes.c_uint64(n), ctypes.c_double(lo), ctypes.c_double(hi),
                              ctypes.c_double(size), a.ctypes.data_as(P), b.ctypes.data_as(P))
    shim.ref_tri_tri_batch(ctypes.c_uint64(n), a.ctypes.data_as(P), b.ctypes.data_as(P), d.ctypes.data_as(P))
    return a, b, d


def tri_tri_ref(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    d = np.zeros(len(a))
    shim.ref_tri_tri_batch(ctypes.c_uint64(len(a)), a.ctypes.data_as(P), b.ctypes.data_as(P), d.ctypes.data_as(P))
    return d


def mindist_ref(a, b):
    d = np.zeros(len(a))
    shim.ref_mindist_aabb_batch(ctypes.c_uint64(len(a)), np.ascontiguousarray(a).ctypes.data_as(P),
                                np.ascontiguousarray(b).ctypes.data_as(P), d.ctypes.data_as(P))
    return d


# Datasets: name -> how to build. Small enough to keep the fixture directory a few MB.
DATASETS = {
    # proj/tests/helpers.hpp mini_dataset(count, spacing, seed, facets, voxel_ratio)
    "mini12_s31": ("mini", 12, 3.4, 31, 100, 0.02),
    "mini10_s61": ("mini", 10, 3.3, 61, 90, 0.02),
    "mini18_s21": ("mini", 18, 3.3, 21, 100, 0.02),
    "mini9_s13_vr15": ("mini", 9, 3.4, 13, 150, 0.15),
    "mini14_s53": ("mini", 14, 3.3, 53, 80, 0.02),
    "mini10_s77": ("mini", 10, 3.2, 77, 90, 0.02),
}
# generated (reference generator + preprocessor, lods [20,60,100]): nuclei vs vessels
GENERATED = {
    "vessels8": dict(shape="tube", facets=300, scale=3.0, count=8, spacing=8.0, jitter=0.3, seed=11),
    "nuclei60": dict(shape="sphere", facets=300, scale=0.35, count=60, seed=12, scatter_in="vessels8"),
    "spheres80a": dict(shape="sphere", facets=120, scale=0.35, count=80, seed=21,
                       scatter_within=(0, 0, 0, 4.0, 4.0, 4.0)),
    "spheres80b": dict(shape="sphere", facets=120, scale=0.35, count=80, seed=22,
                       scatter_within=(0, 0, 0, 4.0, 4.0, 4.0)),
}

# (dataset R, dataset S or "", join kwargs)
JOINS = []
for tau in (0.0, 0.4, 0.9, 1.6, 3.0):   # proj/tests/test_engine.cpp:105-130 sweep
    JOINS.append(("mini18_s21", "", dict(type="within", tau=tau)))
for k in (1, 3):                          # proj/tests/test_engine.cpp:148-178
    JOINS.append(("mini18_s21", "", dict(type="knn", k=k)))
JOINS += [
    ("mini12_s31", "", dict(type="intersect")),
    ("mini12_s31", "", dict(type="within", tau=2.0)),
    ("mini10_s61", "", dict(type="within", tau=1.3)),
    ("mini14_s53", "", dict(type="knn", k=5)),
    ("mini9_s13_vr15", "", dict(type="within", tau=1.2)),
    ("nuclei60", "vessels8", dict(type="within", tau=0.5, lods=[20, 60, 100])),
    ("nuclei60", "vessels8", dict(type="knn", k=3, lods=[20, 60, 100])),
    ("nuclei60", "vessels8", dict(type="intersect", lods=[20, 60, 100])),
    ("spheres80a", "spheres80b", dict(type="intersect", lods=[20, 60, 100])),
    ("spheres80a", "spheres80b", dict(type="within", tau=0.2, lods=[20, 60, 100])),
    ("spheres80a", "", dict(type="within", tau=0.1, lods=[20, 60, 100])),
    # --exact (proj/tests/test_engine.cpp:180-196)
    ("mini10_s77", "", dict(type="within", tau=1.2, exact=True)),
    ("mini14_s53", "", dict(type="knn", k=3, exact=True)),
    ("nuclei60", "vessels8", dict(type="within", tau=0.5, lods=[20, 60, 100], exact=True)),
]

# (dataset, tau, levels) for staged refine-kernel dumps (test_refine.cpp:92-146 logic)
STAGED = [("mini10_s61", 1.4, [20, 40, 60, 80, 100]), ("nuclei60_vs_vessels8", 0.5, [20, 60, 100])]


def build_dataset(name, spec, tmp, built):
    out = os.path.join(HERE, name + ".idx")
    if isinstance(spec, tuple) and spec[0] == "mini":
        _, count, spacing, seed, facets, vr = spec
        rc = shim.ref_mini_dataset(count, ctypes.c_double(spacing), ctypes.c_uint64(seed), facets,
                                   ctypes.c_double(vr), out.encode())
        assert rc == 0, shim.ref_last_error()
        return out, None
    spec = dict(spec)
    d = os.path.join(tmp, name)
    if "scatter_in" in spec:
        ext = built[spec.pop("scatter_in")][1]
        spec["scatter_within"] = tuple(ext)
    gen = ref.generate(d, **spec)
    ref.preprocess(d, out, seed=1, lods=[20, 60, 100])
    return out, gen["extent"]


def main():
    tmp = tempfile.mkdtemp()
    try:
        # ---- geometry vectors
        a, b, d = tri_pairs(42, 2000, -2.0, 2.0, 1.5)
        np.savez(os.path.join(HERE, "tritri_seed42.npz"), a=a, b=b, d=d)
        a, b, d = tri_pairs(20240817, 10000, -2.0, 2.0, 1.5)
        np.savez(os.path.join(HERE, "tritri_seed20240817.npz"), a=a, b=b, d=d)
        # analytic cases (proj/tests/test_geom.cpp:70-93), expected values from the test
        A = [0, 0, 0, 1, 0, 0, 0, 1, 0]
        cases = [
            (A, [0, 0, 0.5, 1, 0, 0.5, 0, 1, 0.5], 0.5),
            (A, [0, 0, 0, 1, 0, 0, 0.5, -1, 1], 0.0),
            (A, [0.25, 0.25, -1, 0.25, 0.25, 1, 3, 3, 1], 0.0),
            (A, [0.25, 0.25, 0.75, 5, 5, 9, -4, 6, 8], 0.75),
            (A, [0.5, -2, 1, 0.5, 2, 1, 0.5, 0, 9], 1.0),
        ]
        ca = np.array([c[0] for c in cases], dtype=np.float64)
        cb = np.array([c[1] for c in cases], dtype=np.float64)
        np.savez(os.path.join(HERE, "tritri_analytic.npz"), a=ca, b=cb, expect=np.array([c[2] for c in cases]),
                 d=tri_tri_ref(ca, cb))
        rng = np.random.default_rng(7)
        lo1 = rng.uniform(-5, 5, (4000, 3))
        lo2 = rng.uniform(-5, 5, (4000, 3))
        b1 = np.concatenate([lo1, lo1 + rng.uniform(0, 3, (4000, 3))], axis=1)
        b2 = np.concatenate([lo2, lo2 + rng.uniform(0, 3, (4000, 3))], axis=1)
        np.savez(os.path.join(HERE, "mindist_random.npz"), a=b1, b=b2, d=mindist_ref(b1, b2))

        # ---- datasets
        built = {}
        for name, spec in DATASETS.items():
            built[name] = build_dataset(name, spec, tmp, built)
        for name, spec in GENERATED.items():
            built[name] = build_dataset(name, spec, tmp, built)

        # ---- joins
        joins = []
        for r, s, kw in JOINS:
            rp = os.path.join(HERE, r + ".idx")
            sp = os.path.join(HERE, s + ".idx") if s else ""
            kw = dict(kw)
            out = ref.join(rp, sp, **kw)
            stages = [{k: v for k, v in st.items() if k != "wall_ms"} for st in out["stats"]["stages"]]
            joins.append({"r": r, "s": s, "kwargs": kw, "records": out["records"], "stages": stages,
                          "query": out["stats"]["query"], "results": out["stats"]["results"]})
        with open(os.path.join(HERE, "joins.json"), "w") as f:
            json.dump(joins, f, indent=0)

        # ---- staged refine-kernel bounds
        for name, tau, levels in STAGED:
            if "_vs_" in name:
                r, s = name.split("_vs_")
            else:
                r, s = name, ""
            rp = os.path.join(HERE, r + ".idx")
            sp = os.path.join(HERE, s + ".idx") if s else ""
            arr = (ctypes.c_uint32 * len(levels))(*levels)
            rc = shim.ref_staged_dump(rp.encode(), sp.encode(), ctypes.c_double(tau), arr, len(levels),
                                      os.path.join(HERE, f"staged_{name}.bin").encode())
            assert rc == 0, shim.ref_last_error()
    finally:
        shutil.rmtree(tmp)
    total = sum(os.path.getsize(os.path.join(HERE, f)) for f in os.listdir(HERE))
    print("golden fixtures:", total / 1e6, "MB")


if __name__ == "__main__":
    main()
