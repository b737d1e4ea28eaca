"""Synthetic benchmark inputs (BASELINE.json configs).

Input tooling, not the join path. Each configuration is the reference generator's
object placement (``generate(..., scatter_within=box)``: object i is centred at a
SplitMix64-drawn target, proj/src/dataset.cpp:183-190, proj/include/trijoin/rng.hpp) applied
to preprocessed template objects (benchdata/*.idx, made by benchdata/make_templates.py
with the reference preprocessor). Object i is template ``i % T`` translated so that its
MBB centre lands on target i (``replicate_index``). The same index files feed the GPU
engine and the reference CPU engine.
"""

import hashlib
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
BENCHDATA = os.path.join(HERE, "..", "benchdata")

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def _splitmix_next(state):
    """Vectorised SplitMix64::next (proj/include/trijoin/rng.hpp:13-18). Mutates state."""
    with np.errstate(over="ignore"):
        state += _GOLDEN
        z = state.copy()
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        return z ^ (z >> np.uint64(31))


def scatter_targets(seed, count, box):
    """Per-object targets of generate(..., scatter_within=box) (dataset.cpp:183-190)."""
    i = np.arange(count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        state = np.uint64(seed) ^ ((i + np.uint64(1)) * _GOLDEN)
    out = np.empty((count, 3), dtype=np.float64)
    for d in range(3):
        u = (_splitmix_next(state) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        lo, hi = float(box[d]), float(box[d + 3])
        out[:, d] = lo + (hi - lo) * u
    return out


def grid_targets(seed, count, spacing, jitter, extent_center):
    """Per-object placement of generate(..., spacing, jitter) on the grid (dataset.cpp:191-200),
    expressed as the target MBB centre (grid shift + the seed mesh's own centre)."""
    per_axis = int(np.ceil(np.cbrt(float(count))))
    i = np.arange(count, dtype=np.int64)
    shift = np.stack([spacing * (i % per_axis), spacing * ((i // per_axis) % per_axis),
                      spacing * (i // (per_axis * per_axis))], axis=1).astype(np.float64)
    if jitter > 0:
        iu = i.astype(np.uint64)
        with np.errstate(over="ignore"):
            state = np.uint64(seed) ^ ((iu + np.uint64(1)) * _GOLDEN)
        for d in range(3):
            u = (_splitmix_next(state) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
            shift[:, d] += -jitter + (2 * jitter) * u
    return shift + np.asarray(extent_center, dtype=np.float64)


# Per configuration: (R spec, S spec or None for self-join, join kwargs). A spec is
# (template file, count, placement) with placement ("scatter", seed, box) or
# ("grid", seed, spacing, jitter).
CONFIGS = {
    # A: within-tau, 1k nuclei x 1k vessels (CPU-runnable reference case)
    "A": (("sphere1000_s035", 1000, ("scatter_in", 12, "V")),
          ("tube1000_s3", 1000, ("grid", 11, 8.0, 0.3)),
          dict(type="within", tau=0.5)),
    # B: intersection, 100k x 100k nuclei on one B200 (the headline N=1 workload)
    "B": (("sphere300_s035", 100000, ("scatter", 21, (0, 0, 0, 41.6, 41.6, 41.6))),
          ("sphere300_s035", 100000, ("scatter", 22, (0, 0, 0, 41.6, 41.6, 41.6))),
          dict(type="intersect")),
    # C: k-NN k=3, 200k nuclei x 10k vessels
    "C": (("sphere300_s035", 200000, ("scatter_in", 32, "V")),
          ("tube1000_s3", 10000, ("grid", 31, 8.0, 0.3)),
          dict(type="knn", k=3)),
    # D: within-tau 0.2, 1M x 1M nuclei
    "D": (("sphere300_s035", 1000000, ("scatter", 41, (0, 0, 0, 100.7, 100.7, 100.7))),
          ("sphere300_s035", 1000000, ("scatter", 42, (0, 0, 0, 100.7, 100.7, 100.7))),
          dict(type="within", tau=0.2)),
    # E: scanned-surface meshes (~20k facets), 50k objects, self-join within tau = 0
    # (scattered in a cube of side 137.5, about 3 MBB neighbours each)
    "E": (("mixed20k", 50000, ("scatter", 53, (0, 0, 0, 137.5, 137.5, 137.5))),
          None,
          dict(type="within", tau=0.0)),
}
LODS = [20, 60, 100]


def _template(name):
    from . import _core
    return _core.load_dataset(os.path.join(BENCHDATA, name + ".idx"))


def _template_centres(tmpl_path):
    """MBB centres of the template objects, read from the 3DPJ1 file headers."""
    import struct
    centres = []
    with open(tmpl_path, "rb") as f:
        data = f.read()
    pos = 5 + 4
    (nl,) = struct.unpack_from("<I", data, pos)
    pos += 4 + 4 * nl
    (n,) = struct.unpack_from("<Q", data, pos)
    pos += 8
    for _ in range(n):
        (blen,) = struct.unpack_from("<Q", data, pos)
        mbb = struct.unpack_from("<6d", data, pos + 8 + 4)
        centres.append([(mbb[0] + mbb[3]) * 0.5, (mbb[1] + mbb[4]) * 0.5, (mbb[2] + mbb[5]) * 0.5])
        pos += 8 + blen
    return np.asarray(centres)


def _placement(spec, count, scale_box, other_extent):
    kind = spec[0]
    if kind == "scatter":
        _, seed, box = spec
        box = np.asarray(box, dtype=np.float64)
        if scale_box != 1.0:
            box = box * scale_box
        return scatter_targets(seed, count, box)
    if kind == "scatter_in":
        _, seed, _ = spec
        return scatter_targets(seed, count, other_extent)
    _, seed, spacing, jitter = spec
    return grid_targets(seed, count, spacing, jitter, (0.0, 0.0, 0.0))


def build_config(name, out_dir, scale=1.0, r_stride=1):
    """Write (r_path, s_path) index files for configuration `name`.

    scale < 1 shrinks object counts by `scale` and scatter boxes by cbrt(scale) (same
    density); r_stride > 1 keeps every r_stride-th query object only (the
    deterministic R-slice used for the CPU baseline; record r' maps back to r' * r_stride).
    Files are cached by a content key.
    """
    from . import _core
    rspec, sspec, _ = CONFIGS[name]
    key = hashlib.sha1(json.dumps([name, scale, r_stride, rspec, sspec], default=str).encode()).hexdigest()[:12]
    os.makedirs(out_dir, exist_ok=True)
    r_path = os.path.join(out_dir, f"{name}_{key}_R.idx")
    s_path = os.path.join(out_dir, f"{name}_{key}_S.idx")
    done = r_path + ".ok"
    if os.path.exists(done):
        if sspec is None:
            return (r_path, s_path) if r_stride > 1 else (s_path, "")
        return r_path, s_path
    box_scale = float(np.cbrt(scale))

    def make(spec, other_extent, stride=1):
        tname, count, placement = spec
        count = max(1, int(round(count * scale)))
        tpath = os.path.join(BENCHDATA, tname + ".idx")
        centres = _template_centres(tpath)
        targets = _placement(placement, count, box_scale, other_extent)
        ids = (np.arange(count) % len(centres)).astype(np.uint32)
        shifts = targets - centres[ids]
        return _core.load_dataset(tpath), ids[::stride], shifts[::stride], targets

    if sspec is None:  # self-join: S is the full R; the R file is a slice of it when r_stride > 1
        tmpl, ids, shifts, _ = make(rspec, None)
        _core.replicate_index(tmpl, s_path, ids.tolist(), shifts.tolist())
        if r_stride > 1:
            _core.replicate_index(tmpl, r_path, ids[::r_stride].tolist(), shifts[::r_stride].tolist())
        else:
            r_path = s_path
        open(done, "w").close()
        return (r_path, s_path) if r_stride > 1 else (s_path, "")
    # S first: the "scatter_in" placements scatter R inside S's extent (generate's
    # scatter_within=V.extent in the reference configurations).
    tmpl_s, ids_s, shifts_s, targets_s = make(sspec, None)
    _core.replicate_index(tmpl_s, s_path, ids_s.tolist(), shifts_s.tolist())
    ext = _dataset_extent(s_path)
    tmpl_r, ids_r, shifts_r, _ = make(rspec, ext, stride=r_stride)
    _core.replicate_index(tmpl_r, r_path, ids_r.tolist(), shifts_r.tolist())
    open(done, "w").close()
    return r_path, s_path


def _dataset_extent(path):
    import struct
    with open(path, "rb") as f:
        data = f.read()
    pos = 5 + 4
    (nl,) = struct.unpack_from("<I", data, pos)
    pos += 4 + 4 * nl
    (n,) = struct.unpack_from("<Q", data, pos)
    pos += 8
    lo = np.full(3, np.inf)
    hi = np.full(3, -np.inf)
    for _ in range(n):
        (blen,) = struct.unpack_from("<Q", data, pos)
        mbb = struct.unpack_from("<6d", data, pos + 8 + 4)
        lo = np.minimum(lo, mbb[:3])
        hi = np.maximum(hi, mbb[3:])
        pos += 8 + blen
    return np.concatenate([lo, hi])


# ---- in-memory inputs (configs whose index files would not fit a disk: D, E) ----

_TEMPLATES = {}


def _template_cached(name):
    if name not in _TEMPLATES:
        _TEMPLATES[name] = _template(name)
    return _TEMPLATES[name]


def _plan(spec, scale, other_extent):
    tname, count, placement = spec
    count = max(1, int(round(count * scale)))
    centres = _template_centres(os.path.join(BENCHDATA, tname + ".idx"))
    targets = _placement(placement, count, float(np.cbrt(scale)), other_extent)
    ids = (np.arange(count) % len(centres)).astype(np.uint32)
    return {"template": tname, "ids": ids, "shifts": np.ascontiguousarray(targets - centres[ids])}


def _template_mbbs(name):
    """Per template object MBB (min.xyz, max.xyz) from the 3DPJ1 file."""
    import struct
    with open(os.path.join(BENCHDATA, name + ".idx"), "rb") as f:
        data = f.read()
    pos = 5 + 4
    (nl,) = struct.unpack_from("<I", data, pos)
    pos += 4 + 4 * nl
    (n,) = struct.unpack_from("<Q", data, pos)
    pos += 8
    out = []
    for _ in range(n):
        (blen,) = struct.unpack_from("<Q", data, pos)
        out.append(struct.unpack_from("<6d", data, pos + 8 + 4))
        pos += 8 + blen
    return np.asarray(out)


def plan_mbbs(plan):
    """MBBs of a plan's objects: the template MBB translated exactly as replicate_* does
    (x -> fl(x + shift) per coordinate)."""
    t = _template_mbbs(plan["template"])[plan["ids"]]
    sh = np.concatenate([plan["shifts"], plan["shifts"]], axis=1)
    return t + sh


def plans_for(name, scale=1.0):
    """{R, S} plans (template name, ids, shifts) of configuration `name`; S is R for a
    self-join. The same objects build_config writes."""
    rspec, sspec, _ = CONFIGS[name]
    if sspec is None:
        p = _plan(rspec, scale, None)
        return {"R": p, "S": p, "self": True}
    ps = _plan(sspec, scale, None)
    m = plan_mbbs(ps)
    ext = np.concatenate([m[:, :3].min(axis=0), m[:, 3:].max(axis=0)])
    return {"R": _plan(rspec, scale, ext), "S": ps, "self": False}


def build_datasets(name, scale=1.0, workers=0):
    """In-memory (R, S, plans) of configuration `name`: the same objects build_config writes,
    replicated straight into memory (_core.replicate_dataset, no index files)."""
    from . import _core
    plans = plans_for(name, scale)
    pr, ps = plans["R"], plans["S"]
    R = _core.replicate_dataset(_template_cached(pr["template"]), pr["ids"], pr["shifts"], workers)
    S = R if plans["self"] else _core.replicate_dataset(_template_cached(ps["template"]), ps["ids"], ps["shifts"],
                                                         workers)
    return R, S, plans


def near_subset(q_mbbs, s_mbbs, tau):
    """Ascending ids of the S objects whose MBB is within tau of some query MBB on every axis
    (a superset of the reference's MBB candidates: mindist <= tau implies every axis gap <= tau)."""
    order = np.argsort(s_mbbs[:, 0], kind="stable")
    smin = s_mbbs[order, 0]
    ext = float(np.max(s_mbbs[:, 3] - s_mbbs[:, 0])) if len(s_mbbs) else 0.0
    keep = np.zeros(len(s_mbbs), dtype=bool)
    for q in q_mbbs:
        lo = np.searchsorted(smin, q[0] - tau - ext, side="left")
        hi = np.searchsorted(smin, q[3] + tau, side="right")
        cand = order[lo:hi]
        c = s_mbbs[cand]
        ok = np.ones(len(cand), dtype=bool)
        for d in range(3):
            gap = np.maximum(c[:, d] - q[3 + d], q[d] - c[:, 3 + d])
            ok &= gap <= tau
        keep[cand[ok]] = True
    return np.nonzero(keep)[0].astype(np.uint32)


def write_slice_files(name, scale, stride, out_dir):
    """Index files for the CPU reference on a deterministic R-slice (every stride-th query) of a
    within-tau configuration, against only the S objects near the slice (near_subset): each
    query's candidates, hence its records, are unchanged (per-query independence),
    and no full-size S file is written. Returns (r_path, s_path, r_ids, s_ids): record (r', s')
    of the slice files is (r_ids[r'], s_ids[s']) of the full join."""
    from . import _core
    plans = plans_for(name, scale)
    tau = float(CONFIGS[name][2].get("tau", 0.0))
    os.makedirs(out_dir, exist_ok=True)
    pr, ps = plans["R"], plans["S"]
    r_ids = np.arange(0, len(pr["ids"]), stride, dtype=np.uint32)
    s_ids = near_subset(plan_mbbs(pr)[r_ids], plan_mbbs(ps), tau)
    key = hashlib.sha1(json.dumps([name, scale, stride]).encode()).hexdigest()[:12]
    r_path = os.path.join(out_dir, f"{name}_{key}_sliceR.idx")
    s_path = os.path.join(out_dir, f"{name}_{key}_sliceS.idx")
    _core.replicate_index(_template_cached(pr["template"]), r_path, pr["ids"][r_ids].tolist(),
                          pr["shifts"][r_ids].tolist())
    _core.replicate_index(_template_cached(ps["template"]), s_path, ps["ids"][s_ids].tolist(),
                          ps["shifts"][s_ids].tolist())
    return r_path, s_path, r_ids, s_ids
