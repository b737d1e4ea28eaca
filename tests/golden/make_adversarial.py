"""Adversarial culling fixtures (tests/golden/adv_*.idx + adversarial_joins.json), made by the
reference itself.

TEST INFRASTRUCTURE. Runs only in the build container (needs oracle/_ref, the reference
trijoin built from /root/reference/proj by oracle/Makefile). The meshes are built here as OFF
text; indexing (trijoin.preprocess) and every expected record / stage counter
(trijoin.join) come from the reference's own code.

The product's exact-preserving culling (csrc/refine_kernel.cuh) rests on hand-set margins:
the rounding margin delta = 1e-5 (B + L_i + L_j) + 1e-12 M, the separating-axis margin
8e-6 R, the plane clearance 3.2e-5 R, the 1e-2 sine cut for well-shaped facets, the DP4A
conditioning threshold and the reference's own spurious-piercing regime. These fixtures put
facet pairs right at those edges:

  adv_faces_R / adv_faces_S   box slabs around coordinate 100 whose faces are parallel or
                              tilted by 1e-7 .. 2e-2 rad, at gaps 0 .. 1e-2 (and slight
                              interpenetration); many facet pairs with nearly parallel
                              edge / plane combinations and distances down to 1e-12
  adv_slivers                 long thin bars (aspect 60 .. 200, triangles with sin ~ 5e-3 ..
                              1.7e-2, straddling the 1e-2 cut) crossed at small angles and
                              near-touching, around coordinate 100 (self-join)
  adv_edges_R / adv_edges_S   bars whose long edges run nearly parallel (1e-6 .. 1e-2 rad)
                              at gaps 1e-10 .. 1e-3 around coordinate -100

    python tests/golden/make_adversarial.py
"""
import json
import math
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
import trijoin as ref  # noqa: E402

LODS = [20, 60, 100]


def box_mesh(size, cells):
    """Closed, outward-oriented triangulated box [0, sx] x [0, sy] x [0, sz] with cells[d] grid
    cells along axis d (every face quad split along one diagonal)."""
    size = np.asarray(size, dtype=np.float64)
    n = np.asarray(cells, dtype=np.int64)
    index = {}
    verts = []

    def vid(i, j, k):
        key = (i, j, k)
        if key not in index:
            index[key] = len(verts)
            verts.append([size[0] * i / n[0], size[1] * j / n[1], size[2] * k / n[2]])
        return index[key]

    facets = []
    # faces: axis a fixed at 0 or n[a]; the other two axes (u, v) span the face
    for a in range(3):
        u, v = (a + 1) % 3, (a + 2) % 3
        for side in (0, 1):
            for iu in range(n[u]):
                for iv in range(n[v]):
                    def p(du, dv):
                        c = [0, 0, 0]
                        c[a] = side * n[a]
                        c[u] = iu + du
                        c[v] = iv + dv
                        return vid(*c)
                    q = [p(0, 0), p(1, 0), p(1, 1), p(0, 1)]
                    if side == 0:  # outward normal -a: reverse the (u, v) winding
                        q = q[::-1]
                    facets.append([q[0], q[1], q[2]])
                    facets.append([q[0], q[2], q[3]])
    return np.asarray(verts), np.asarray(facets)


def rot(axis, angle):
    axis = np.asarray(axis, dtype=np.float64)
    axis = axis / np.linalg.norm(axis)
    k = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + math.sin(angle) * k + (1 - math.cos(angle)) * (k @ k)


def write_off(path, verts, facets):
    with open(path, "w") as f:
        f.write(f"OFF\n{len(verts)} {len(facets)} 0\n")
        for v in verts:
            f.write("%.17g %.17g %.17g\n" % tuple(v))
        for t in facets:
            f.write("3 %d %d %d\n" % tuple(t))


def emit(objects, out_idx, tmp):
    d = tempfile.mkdtemp(dir=tmp)
    for i, (v, t) in enumerate(objects):
        write_off(os.path.join(d, f"{i:04d}.off"), v, t)
    n = ref.preprocess(d, out_idx, seed=1, lods=LODS)
    assert n == len(objects)


# Every pair is finally turned by a generic rotation about its contact region, so the
# objects' axis-aligned MBBs overlap deeply while the surfaces stay `gap` apart: the MBB and
# voxel stages cannot settle these pairs and the facet refinement has to.

def turned(v, centre, q):
    return (v - centre) @ q.T + centre


def faces_family():
    """Slab pairs: S slab above R slab, the facing faces parallel or tilted, gap g."""
    R, S = [], []
    gaps = [0.0, 1e-12, 1e-10, 1e-8, 1e-6, 1e-4, 1e-2, -1e-6]
    tilts = [0.0, 1e-7, 1e-5, 1e-3, 2e-2]
    base = np.array([100.0, 100.0, 100.0])
    k = 0
    for g in gaps:
        for t in tilts:
            v, f = box_mesh((1.0, 1.0, 0.3), (6, 6, 2))
            o = base + np.array([3.0 * (k % 8), 3.0 * (k // 8), 0.0])
            R.append((v + o, f))
            w, f2 = box_mesh((1.0, 1.0, 0.3), (5, 7, 2))  # different grid: facets not aligned
            c = np.array([0.5, 0.5, 0.0])
            w = (w - c) @ rot((1.0, 0.3, 0.0), t).T + c
            # lowest point of the tilted slab at height 0.3 + g above R's base plane
            w[:, 2] += 0.3 + g - w[:, 2].min()
            w[:, 0] += 0.05 * (k % 3)  # shifted in x: partial overlap of the faces
            q = rot((1.0, 2.0, 3.0), 0.4 + 0.1 * (k % 5))
            centre = np.array([0.5, 0.5, 0.3])
            R[-1] = (turned(v, centre, q) + o, f)
            S.append((turned(w, centre, q) + o, f2))
            k += 1
    return R, S


def bar(length, width, cells_long, axis_rot, angle, offset):
    v, f = box_mesh((length, width, width), (cells_long, 1, 1))
    c = np.array([length / 2, width / 2, width / 2])
    v = (v - c) @ rot(axis_rot, angle).T + offset
    return v, f


def slivers_family():
    """Thin bars (sliver side triangles) crossing / touching at small angles (self-join)."""
    objs = []
    base = np.array([100.0, 101.0, 99.0])
    aspects = [(6.0, 0.03, 1), (6.0, 0.06, 1), (6.0, 0.1, 2), (6.0, 0.1, 1)]  # sin ~ 5e-3 .. 1.7e-2
    k = 0
    for length, width, cl in aspects:
        for ang, gap in [(0.0, 1e-9), (1e-3, 0.0), (2e-2, 1e-6), (math.pi / 2, 1e-12), (5e-3, -1e-7)]:
            o = base + np.array([0.0, 8.0 * (k % 5), 1.5 * (k // 5)])
            objs.append(bar(length, width, cl * 20, (0, 0, 1), 0.0, o))
            # partner bar on top, rotated about z by ang, touching at gap
            o2 = o + np.array([0.3, 0.0, width + gap])
            objs.append(bar(length, width, cl * 20 + 1, (0, 0, 1), ang, o2))
            q = rot((2.0, -1.0, 1.0), 0.5 + 0.15 * (k % 4))
            centre = o + np.array([0.15, 0.0, width / 2])
            objs[-2] = (turned(objs[-2][0], centre, q), objs[-2][1])
            objs[-1] = (turned(objs[-1][0], centre, q), objs[-1][1])
            k += 1
    return objs


def edges_family():
    """Bars whose long edges run nearly parallel at tiny gaps (edge-edge configurations)."""
    R, S = [], []
    base = np.array([-100.0, -100.0, -100.0])
    k = 0
    for ang in [0.0, 1e-6, 1e-4, 1e-2]:
        for gap in [1e-10, 1e-7, 1e-5, 1e-3]:
            o = base + np.array([0.0, 4.0 * (k % 4), 4.0 * (k // 4)])
            # R bar rotated 45 deg about its long axis: its top is an edge
            R.append(bar(4.0, 0.2, 30, (1, 0, 0), math.pi / 4, o))
            v, f = bar(4.0, 0.2, 27, (1, 0, 0), math.pi / 4, np.zeros(3))
            v = v @ rot((0, 0, 1), ang).T
            # S bar's lowest edge `gap` above R's highest edge
            v[:, 2] += (R[-1][0][:, 2].max() - o[2]) + gap - v[:, 2].min()
            q = rot((1.0, 1.0, -2.0), 0.6 + 0.1 * (k % 3))
            top = np.array([0.0, 0.0, R[-1][0][:, 2].max()])
            R[-1] = (turned(R[-1][0], top, q), R[-1][1])
            S.append((turned(v + o, top, q), f))
            k += 1
    return R, S


DATASETS = {}
JOINS = []


def main():
    tmp = tempfile.mkdtemp()
    try:
        fr, fs = faces_family()
        emit(fr, os.path.join(HERE, "adv_faces_R.idx"), tmp)
        emit(fs, os.path.join(HERE, "adv_faces_S.idx"), tmp)
        emit(slivers_family(), os.path.join(HERE, "adv_slivers.idx"), tmp)
        er, es = edges_family()
        emit(er, os.path.join(HERE, "adv_edges_R.idx"), tmp)
        emit(es, os.path.join(HERE, "adv_edges_S.idx"), tmp)
        joins = []
        cases = []
        for r, s in (("adv_faces_R", "adv_faces_S"), ("adv_slivers", ""), ("adv_edges_R", "adv_edges_S")):
            cases.append((r, s, dict(type="intersect", lods=LODS)))
            for tau in (1e-11, 1e-9, 1e-7, 1e-5, 1e-3, 0.05):
                cases.append((r, s, dict(type="within", tau=tau, lods=LODS)))
            cases.append((r, s, dict(type="knn", k=2, lods=LODS)))
            cases.append((r, s, dict(type="within", tau=1e-6, lods=LODS, exact=True)))
        for r, s, kw in cases:
            rp = os.path.join(HERE, r + ".idx")
            sp = os.path.join(HERE, s + ".idx") if s else ""
            out = ref.join(rp, sp, **kw)
            stages = [{k: v for k, v in st.items() if k != "wall_ms"} for st in out["stats"]["stages"]]
            joins.append({"r": r, "s": s, "kwargs": kw, "records": out["records"], "stages": stages,
                          "query": out["stats"]["query"], "results": out["stats"]["results"]})
            print(r, s, kw, "results", out["stats"]["results"],
                  "facet pairs", sum(st["facet_pairs"] for st in out["stats"]["stages"]))
        with open(os.path.join(HERE, "adversarial_joins.json"), "w") as f:
            json.dump(joins, f, indent=0)
    finally:
        shutil.rmtree(tmp)


if __name__ == "__main__":
    main()
