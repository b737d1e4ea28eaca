"""Golden vectors for the geometric primitives and the exhaustive oracle join, from the
reference itself.

TEST INFRASTRUCTURE. Runs only in the build container (needs oracle/_ref: the reference
trijoin built from /root/reference/proj by oracle/Makefile). Every expected value is an
output of the reference's own code:
  * primitives.npz: point_segment_distance, point_triangle_distance, segment_segment_distance
    (proj/src/geom.cpp:18-113) through oracle/ref_shim.cpp on the analytic cases of
    proj/tests/test_geom.cpp:36-68 plus seeded random and degenerate inputs (zero-length and
    parallel segments, collinear and coincident-vertex triangles, points on edges / in the
    plane, coordinates ~1e2);
  * oracle_joins.json: the reference trijoin.oracle (proj/src/oracle.cpp:124-186) records on
    the golden datasets (within tau sweep, intersect, k-NN).

    python tests/golden/make_primitives.py
"""
import ctypes
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
import trijoin as ref  # noqa: E402

P = ctypes.POINTER(ctypes.c_double)
shim = ctypes.CDLL(os.path.join(ROOT, "oracle", "_ref", "libref_shim.so"))


def call(fn, a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    d = np.zeros(len(a))
    getattr(shim, fn)(ctypes.c_uint64(len(a)), a.ctypes.data_as(P), b.ctypes.data_as(P), d.ctypes.data_as(P))
    return d


def degenerate_tris(rng, n, scale):
    """Collinear, coincident-vertex and sliver triangles."""
    out = []
    for i in range(n):
        p = rng.uniform(-scale, scale, 3)
        d = rng.uniform(-1, 1, 3)
        kind = i % 4
        if kind == 0:  # collinear
            out.append(np.concatenate([p, p + d, p + 2.5 * d]))
        elif kind == 1:  # two coincident vertices
            out.append(np.concatenate([p, p, p + d]))
        elif kind == 2:  # all coincident
            out.append(np.concatenate([p, p, p]))
        else:  # sliver near the degeneracy threshold
            e = rng.uniform(-1, 1, 3) * 1e-13
            out.append(np.concatenate([p, p + d, p + 0.5 * d + e]))
    return np.array(out)


def main():
    rng = np.random.default_rng(20261017)
    out = {}
    # ---- point_segment_distance
    pts = [[0.5, 1, 0], [-1, 0, 0], [3, 0, 0], [0.25, 0, 0], [1, 1, 1]]
    segs = [[0, 0, 0, 1, 0, 0]] * 4 + [[1, 1, 1, 1, 1, 1]]
    n = 6000
    p = rng.uniform(-3, 3, (n, 3))
    s = np.concatenate([rng.uniform(-3, 3, (n, 3)), rng.uniform(-3, 3, (n, 3))], axis=1)
    s[::7, 3:] = s[::7, :3]  # zero-length segments
    p[::11] = s[::11, :3] + 0.37 * (s[::11, 3:] - s[::11, :3])  # points on the segment
    big = rng.uniform(95, 105, (1000, 9))
    ps_a = np.concatenate([np.array(pts, float), p, big[:, :3]])
    ps_b = np.concatenate([np.array(segs, float), s, big[:, 3:]])
    out["ps_a"], out["ps_b"], out["ps_d"] = ps_a, ps_b, call("ref_point_segment_batch", ps_a, ps_b)
    # ---- point_triangle_distance (test_geom.cpp:48-58 analytic + random + degenerate)
    t = [0, 0, 0, 2, 0, 0, 0, 2, 0]
    line = [0, 0, 0, 1, 0, 0, 2, 0, 0]
    an_p = [[0.5, 0.5, 3.0], [0.5, 0.5, 0.0], [-1, -1, 0], [3, 3, 0], [1, 1, 0]]
    an_t = [t, t, t, t, line]
    base = rng.uniform(-2, 2, (n, 3))
    tris = np.concatenate([base, base + rng.uniform(-1.5, 1.5, (n, 3)), base + rng.uniform(-1.5, 1.5, (n, 3))],
                          axis=1)
    q = rng.uniform(-3, 3, (n, 3))
    # points in the triangle's plane / on its edges / at its vertices
    w = rng.uniform(0, 1, (n, 2))
    inplane = tris[:, :3] + w[:, :1] * (tris[:, 3:6] - tris[:, :3]) + w[:, 1:] * (tris[:, 6:] - tris[:, :3])
    q[::5] = inplane[::5]
    q[1::13] = tris[1::13, 3:6]
    q[2::17] = 0.5 * (tris[2::17, :3] + tris[2::17, 6:])
    dg = degenerate_tris(rng, 2000, 2.0)
    dq = rng.uniform(-3, 3, (2000, 3))
    bt = 100.0 + rng.uniform(-1, 1, (1000, 9))
    bq = 100.0 + rng.uniform(-1.5, 1.5, (1000, 3))
    pt_a = np.concatenate([np.array(an_p, float), q, dq, bq])
    pt_b = np.concatenate([np.array(an_t, float), tris, dg, bt])
    out["pt_a"], out["pt_b"], out["pt_d"] = pt_a, pt_b, call("ref_point_triangle_batch", pt_a, pt_b)
    # ---- segment_segment_distance (test_geom.cpp:60-68 analytic + random + degenerate)
    an_a = [[0, 0, 0, 1, 0, 0]] * 3 + [[0, 0, 0, 0, 0, 0]]
    an_b = [[0.5, -1, 0, 0.5, 1, 0], [0, 1, 0, 1, 1, 0], [2, 0, 1, 2, 0, -1], [1, 1, 1, 1, 1, 1]]
    sa = rng.uniform(-2, 2, (n, 6))
    sb = rng.uniform(-2, 2, (n, 6))
    d1 = sa[:, 3:] - sa[:, :3]
    sb[::3, 3:] = sb[::3, :3] + d1[::3] * rng.uniform(-2, 2, (len(sb[::3]), 1))  # parallel
    sb[1::9, 3:] = sb[1::9, :3]  # point-degenerate b
    sa[2::9, 3:] = sa[2::9, :3]  # point-degenerate a
    sb[4::10] = sa[4::10] + np.array([0.1, 0.0, 0.0, 0.1, 0.0, 0.0])  # shifted copies (collinear-ish)
    bs_a = 100.0 + rng.uniform(-1, 1, (1000, 6))
    bs_b = 100.0 + rng.uniform(-1, 1, (1000, 6))
    ss_a = np.concatenate([np.array(an_a, float), sa, bs_a])
    ss_b = np.concatenate([np.array(an_b, float), sb, bs_b])
    out["ss_a"], out["ss_b"], out["ss_d"] = ss_a, ss_b, call("ref_segment_segment_batch", ss_a, ss_b)
    # ---- tri_tri over degenerate triangles (the engine goldens cover regular ones)
    da = degenerate_tris(rng, 2000, 1.0)
    db = np.concatenate([degenerate_tris(rng, 1000, 1.0), rng.uniform(-1, 1, (1000, 9))])
    out["tt_a"], out["tt_b"], out["tt_d"] = da, db, call("ref_tri_tri_batch", da, db)
    np.savez_compressed(os.path.join(HERE, "primitives.npz"), **out)

    # ---- exhaustive oracle joins (reference trijoin.oracle)
    cases = [
        ("mini18_s21", "", dict(type="within", tau=0.0)),
        ("mini18_s21", "", dict(type="within", tau=0.9)),
        ("mini18_s21", "", dict(type="within", tau=3.0)),
        ("mini18_s21", "", dict(type="knn", k=1)),
        ("mini18_s21", "", dict(type="knn", k=3)),
        ("mini12_s31", "", dict(type="intersect")),
        ("mini10_s61", "", dict(type="within", tau=1.3)),
        ("mini14_s53", "", dict(type="knn", k=5)),
        ("nuclei60", "vessels8", dict(type="within", tau=0.5)),
        ("nuclei60", "vessels8", dict(type="knn", k=3)),
        ("spheres80a", "spheres80b", dict(type="intersect")),
        ("spheres80a", "spheres80b", dict(type="knn", k=40)),
    ]
    res = []
    for r, s, kw in cases:
        rp = os.path.join(HERE, r + ".idx")
        sp = os.path.join(HERE, s + ".idx") if s else ""
        o = ref.oracle(rp, sp, workers=4, **kw)
        recs = [[x[0], x[1], float(x[2]).hex(), float(x[3]).hex(), x[4], x[5]] for x in o["records"]]
        st = [{k: v for k, v in x.items() if k != "wall_ms"} for x in o["stats"]["stages"]]
        res.append({"r": r, "s": s, "kw": kw, "records": recs, "stages": st})
        print(r, s, kw, len(recs))
    with open(os.path.join(HERE, "oracle_joins.json"), "w") as f:
        json.dump(res, f, indent=0)


if __name__ == "__main__":
    main()
