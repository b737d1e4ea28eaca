#!/usr/bin/env python3
"""Offline preprocessing throughput: the GPU hd / ph fill and k-means
voxelisation (tj_facet_hd_batch / tj_facet_ph_batch / tj_voxelize_batch) against the reference's
own CPU code (oracle/_ref: compute_facet_hd through its TriBvh, build_lod_ladder, voxelize), on
E-style "scanned" meshes (~20k facets, radial noise), lods [20, 60, 100], hd_grid 8.

The reference ladders (simplifier + hd / ph) are built once on the CPU; the GPU recomputes every
coarse level's hd and ph and the coarsest level's voxel labels, checked bitwise against them.
CPU rate: compute_facet_hd over the same facets, one object per host thread, all cores.

    python scripts/bench_preprocess.py [--objects 16] [--facets 20000]
"""
import argparse
import ctypes
import json
import os
import sys
import tempfile
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import tjtest  # noqa: E402
import make_preprocess as mp  # noqa: E402  (reference probes: ladder / facet_hd / voxelize)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--objects", type=int, default=16)
    ap.add_argument("--facets", type=int, default=20000)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    rng = np.random.default_rng(7)
    meshes, ladders = [], []
    t0 = time.perf_counter()
    for i in range(a.objects):
        v, f = mp.gen_mesh("sphere", a.facets, 5.0, 100 + i)
        v = v * (1.0 + 0.03 * rng.standard_normal((len(v), 1))) + rng.uniform(0, 100, 3)
        meshes.append((v, f))
    with ThreadPoolExecutor(os.cpu_count()) as ex:
        ladders = list(ex.map(lambda m: mp.ladder(m[0], m[1], [20, 60, 100], 8), meshes))
    t_ladder = time.perf_counter() - t0
    # work: every coarse-level facet (hd: 45 point-to-mesh queries each; ph: its originals)
    ms, qs, want_hd, want_ph, ancs = [], [], [], [], []  # per (object, coarse level)
    for (v, f), L in zip(meshes, ladders):
        for li in (0, 1):
            ms.append((v, f))
            qs.append(L[li]["verts"][L[li]["facets"]].reshape(-1, 9))
            want_hd.append(L[li]["hd"])
            want_ph.append(L[li]["ph"])
            ancs.append(L[li]["anc"])
    # hd: one tree per object, queried by both coarse levels' facets
    hd_ms = meshes
    hd_qs = [np.concatenate([qs[2 * i], qs[2 * i + 1]]) for i in range(len(meshes))]
    n_q = sum(len(q) for q in qs)
    capi = tjtest.Capi()
    capi.facet_hd(hd_ms[:1], hd_qs[:1], 8)  # warm-up (context, kernels)
    gpu_hd_s, gpu_ph_s, gpu_vox_s = [], [], []
    for _ in range(a.reps):
        t = time.perf_counter()
        hd = capi.facet_hd(hd_ms, hd_qs, 8)
        gpu_hd_s.append(time.perf_counter() - t)
        t = time.perf_counter()
        ph = capi.facet_ph(ms, qs, ancs)
        gpu_ph_s.append(time.perf_counter() - t)
        coarse = [(L[0]["verts"], L[0]["facets"]) for L in ladders]
        ks = [int(np.ceil(0.02 * len(m[1]))) for m in meshes]
        seeds = [(0 ^ ((i + 1) * 0x9E3779B97F4A7C15)) % (1 << 64) for i in range(len(meshes))]
        t = time.perf_counter()
        labels = capi.voxelize(coarse, ks, seeds)
        gpu_vox_s.append(time.perf_counter() - t)
    hd_ok = bool((tjtest.bits(hd) == tjtest.bits(np.concatenate(want_hd))).all())
    ph_ok = bool((tjtest.bits(ph) == tjtest.bits(np.concatenate(want_ph))).all())
    ref_labels = [mp.voxelize(c[0], c[1], k, s) for c, k, s in zip(coarse, ks, seeds)]
    vox_ok = all((x == y).all() for x, y in zip(labels, ref_labels))
    # reference CPU: compute_facet_hd over the same facets, one mesh-level per thread, all cores
    cores = os.cpu_count()
    t = time.perf_counter()
    with ThreadPoolExecutor(cores) as ex:
        ref_hd = list(ex.map(lambda mq: mp.facet_hd(mq[0][0], mq[0][1], mq[1], 8), zip(ms, qs)))
    cpu_hd_s = time.perf_counter() - t
    cpu_ok = bool((tjtest.bits(np.concatenate(ref_hd)) == tjtest.bits(np.concatenate(want_hd))).all())
    line = {
        "metric": "hd facets/s (compute_facet_hd, 45 point-to-mesh queries per facet)",
        "workload": f"{a.objects} noisy spheres x {a.facets} facets, coarse levels 20/60, hd_grid 8",
        "facets": n_q, "gpu_hd_s": min(gpu_hd_s), "gpu_hd_facets_per_s": n_q / min(gpu_hd_s),
        "gpu_ph_s": min(gpu_ph_s), "gpu_voxelize_s": min(gpu_vox_s),
        "cpu_hd_s": cpu_hd_s, "cpu_hd_facets_per_s": n_q / cpu_hd_s, "cpu_cores": cores, "cpu_kind": "reference",
        "speedup_hd": cpu_hd_s / min(gpu_hd_s),
        "parity": {"hd_bitwise": hd_ok, "ph_bitwise": ph_ok, "voxelize_equal": vox_ok, "cpu_hd_equals_ladder": cpu_ok},
        "ref_ladder_build_s": t_ladder,
        "note": "GPU times include the host->device copy of the meshes and queries and the result copy back",
    }
    print(json.dumps(line))
    return 0 if hd_ok and ph_ok and vox_ok else 1


if __name__ == "__main__":
    sys.exit(main())
