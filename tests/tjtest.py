"""Test helpers: ctypes bindings of the product C-ABI (include/tj_capi.h), the C restatement
oracle (oracle/tj_oracle.c) and the reference probes (oracle/ref_shim.cpp), plus golden
fixture access. Only tests import this module."""
import ctypes
import json
import os
import re
import struct

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
GOLDEN = os.path.join(ROOT, "tests", "golden")
LIB = os.path.join(ROOT, "paper_2604_19982_b200", "libtrijoin_b200.so")
ORACLE_LIB = os.path.join(ROOT, "oracle", "_ref", "libtj_oracle.so")
SHIM_LIB = os.path.join(ROOT, "oracle", "_ref", "libref_shim.so")
REF_PKG = os.path.join(ROOT, "oracle", "_ref")

PD = ctypes.POINTER(ctypes.c_double)
PU64 = ctypes.POINTER(ctypes.c_uint64)
PU32 = ctypes.POINTER(ctypes.c_uint32)

STAGE_NAMES = {-3: "undecided", -2: "mbb", -1: "voxel", 100: "exact"}


def stage_name(code):
    return STAGE_NAMES.get(code, f"lod-{code}")


def ptr(a, t=PD):
    return a.ctypes.data_as(t)


# ---------------------------------------------------------------- product C-ABI
class DatasetView(ctypes.Structure):
    _fields_ = [("n_objects", ctypes.c_uint32), ("n_levels", ctypes.c_uint32),
                ("levels", ctypes.POINTER(ctypes.c_int32)), ("mbb", PD), ("anchor", PD), ("voxel_offsets", PU64),
                ("voxel_box", PD), ("voxel_anchor", PD), ("facet_offsets", ctypes.POINTER(PU64)),
                ("facets", ctypes.POINTER(PD))]


class JoinSpec(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int32), ("tau", ctypes.c_double), ("k", ctypes.c_uint32),
                ("filter_chunk", ctypes.c_uint64), ("refine_chunk", ctypes.c_uint64), ("n_lods", ctypes.c_uint32),
                ("lods", PU32), ("pipeline", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("shard_index", ctypes.c_uint32), ("shard_count", ctypes.c_uint32), ("shard_block", ctypes.c_uint32)]


MAXL = 16


class MeshSetView(ctypes.Structure):
    _fields_ = [("n_objects", ctypes.c_uint32), ("tri_offsets", PU64), ("tris", PD)]


class ExhaustiveResult(ctypes.Structure):
    _fields_ = [("n_records", ctypes.c_uint64), ("r", PU32), ("s", PU32), ("d", PD), ("rank", PU32),
                ("object_pairs", ctypes.c_uint64), ("facet_pairs_evaluated", ctypes.c_uint64),
                ("total_ms", ctypes.c_double)]


class JoinResult(ctypes.Structure):
    _fields_ = [("n_cands", ctypes.c_uint64), ("n_queries", ctypes.c_uint32), ("pair_r", PU32), ("pair_s", PU32),
                ("lb", PD), ("ub", PD), ("status", ctypes.POINTER(ctypes.c_uint8)),
                ("decided_at", ctypes.POINTER(ctypes.c_int16)), ("r2op_offsets", PU64), ("num_confirmed", PU32),
                ("vp_generated", ctypes.c_uint64), ("vp_pruned", ctypes.c_uint64),
                ("filter_chunks", ctypes.c_uint64), ("oversized_chunks", ctypes.c_uint64),
                ("n_levels_run", ctypes.c_uint32), ("level", ctypes.c_uint32 * MAXL),
                ("level_vps", ctypes.c_uint64 * MAXL), ("level_facet_pairs", ctypes.c_uint64 * MAXL),
                ("level_pairs_evaluated", ctypes.c_uint64 * MAXL), ("level_pairs_tested", ctypes.c_uint64 * MAXL),
                ("level_ms", ctypes.c_double * MAXL), ("level_kernel_ms", ctypes.c_double * MAXL),
                ("refine_chunks", ctypes.c_uint64), ("mbb_ms", ctypes.c_double), ("voxel_ms", ctypes.c_double),
                ("refine_ms", ctypes.c_double), ("total_ms", ctypes.c_double),
                ("level_pairs_screened", ctypes.c_uint64 * MAXL),
                ("level_pairs_verified", ctypes.c_uint64 * MAXL),
                ("level_vps_skipped", ctypes.c_uint64 * MAXL),
                ("level_facets_dropped", ctypes.c_uint64 * MAXL),
                ("level_wait_ms", ctypes.c_double * MAXL), ("decision_mode", ctypes.c_int32),
                ("queue_reruns", ctypes.c_uint32), ("mat_chunks", ctypes.c_uint64),
                ("level_screen_ms", ctypes.c_double * MAXL)]


def capi_functions():
    """Function names declared in include/tj_capi.h."""
    with open(os.path.join(ROOT, "include", "tj_capi.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tj_[a-z0-9_]+)\s*\(", text)))


def load_capi():
    lib = ctypes.CDLL(LIB)
    lib.tj_last_error.restype = ctypes.c_char_p
    lib.tj_global_last_error.restype = ctypes.c_char_p
    lib.tj_host_dataset_view.restype = ctypes.POINTER(DatasetView)
    lib.tj_host_dataset_bytes.restype = ctypes.c_uint64
    lib.tj_kernel_launches.restype = ctypes.c_uint64
    lib.tj_dataset_device_bytes.restype = ctypes.c_uint64
    return lib


class Capi:
    """Thin RAII-ish wrapper used by the GPU parity tests (calls go through the C-ABI)."""

    TYPES = {"within": 0, "intersect": 1, "knn": 2}

    def __init__(self, device=0):
        self.lib = load_capi()
        self.ctx = ctypes.c_void_p()
        rc = self.lib.tj_ctx_create(device, ctypes.byref(self.ctx))
        if rc != 0:
            raise RuntimeError(self.lib.tj_global_last_error().decode())

    def err(self):
        return self.lib.tj_last_error(self.ctx).decode()

    def check(self, rc):
        if rc != 0:
            raise RuntimeError(f"C-ABI status {rc}: {self.err()}")

    def tri_tri(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = np.zeros(len(a))
        self.check(self.lib.tj_tri_tri_batch(self.ctx, ctypes.c_uint64(len(a)), ptr(a), ptr(b), ptr(out)))
        return out

    def mindist(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = np.zeros(len(a))
        self.check(self.lib.tj_mindist_batch(self.ctx, ctypes.c_uint64(len(a)), ptr(a), ptr(b), ptr(out)))
        return out

    GEOM = {"mindist": 0, "point_segment": 1, "point_triangle": 2, "segment_segment": 3, "tri_tri": 4}

    def geom(self, op, a, b):
        """tj_geom_batch (include/tj_capi.h): out[i] = op(a[i], b[i])."""
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = np.zeros(len(a))
        self.check(self.lib.tj_geom_batch(self.ctx, ctypes.c_int32(self.GEOM[op]), ctypes.c_uint64(len(a)), ptr(a),
                                          ptr(b), ptr(out)))
        return out

    @staticmethod
    def mesh_set(meshes):
        """Pack [(verts f64[nv, 3], facets u32[nf, 3]), ...] into the C-ABI mesh-set arrays."""
        vo = np.zeros(len(meshes) + 1, dtype=np.uint64)
        fo = np.zeros(len(meshes) + 1, dtype=np.uint64)
        for i, (v, f) in enumerate(meshes):
            vo[i + 1] = vo[i] + len(v)
            fo[i + 1] = fo[i] + len(f)
        v = np.ascontiguousarray(np.concatenate([np.asarray(m[0], np.float64).reshape(-1, 3) for m in meshes]))
        f = np.ascontiguousarray(np.concatenate([np.asarray(m[1], np.uint32).reshape(-1, 3) for m in meshes]))
        return vo, v, fo, f

    def facet_hd(self, meshes, queries, grid=8):
        """tj_facet_hd_batch: queries[i] (f64[n, 9]) against original mesh meshes[i]."""
        vo, v, fo, f = self.mesh_set(meshes)
        qo = np.zeros(len(meshes) + 1, dtype=np.uint64)
        for i, q in enumerate(queries):
            qo[i + 1] = qo[i] + len(q)
        q = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float64).reshape(-1, 9) for x in queries]))
        out = np.zeros(int(qo[-1]))
        self.check(self.lib.tj_facet_hd_batch(self.ctx, ctypes.c_uint32(len(meshes)), ptr(vo, PU64), ptr(v),
                                              ptr(fo, PU64), ptr(f, PU32), ptr(qo, PU64), ptr(q),
                                              ctypes.c_int32(grid), ptr(out)))
        return out

    def facet_ph(self, meshes, lods, ancestors):
        """tj_facet_ph_batch: ph of every facet of lods[i] (f64[n, 9]) from original mesh
        meshes[i] with ancestors[i] (u32 per original facet)."""
        vo, v, fo, f = self.mesh_set(meshes)
        lo = np.zeros(len(meshes) + 1, dtype=np.uint64)
        for i, q in enumerate(lods):
            lo[i + 1] = lo[i] + len(q)
        lt = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float64).reshape(-1, 9) for x in lods]))
        anc = np.ascontiguousarray(np.concatenate([np.asarray(a, np.uint32) for a in ancestors]))
        out = np.zeros(int(lo[-1]))
        self.check(self.lib.tj_facet_ph_batch(self.ctx, ctypes.c_uint32(len(meshes)), ptr(vo, PU64), ptr(v),
                                              ptr(fo, PU64), ptr(f, PU32), ptr(anc, PU32), ptr(lo, PU64), ptr(lt),
                                              ptr(out)))
        return out

    def voxelize(self, meshes, k, seeds):
        """tj_voxelize_batch: labels per facet of each (coarsest-level) mesh."""
        vo, v, fo, f = self.mesh_set(meshes)
        kk = np.ascontiguousarray(k, dtype=np.uint32)
        ss = np.ascontiguousarray(seeds, dtype=np.uint64)
        out = np.zeros(int(fo[-1]), dtype=np.uint32)
        self.check(self.lib.tj_voxelize_batch(self.ctx, ctypes.c_uint32(len(meshes)), ptr(vo, PU64), ptr(v),
                                              ptr(fo, PU64), ptr(f, PU32), ptr(kk, PU32), ptr(ss, PU64), ptr(out, PU32)))
        return [out[int(fo[i]):int(fo[i + 1])] for i in range(len(meshes))]

    def exhaustive(self, R, S, type="within", tau=0.0, k=1):
        """tj_exhaustive_join over level-100 triangle sets given as (tri_offsets u64[n+1],
        tris f64[m, 9]); S None = self-join. Returns a list of (r, s, d, rank)."""
        def view(ms):
            off = np.ascontiguousarray(ms[0], dtype=np.uint64)
            tris = np.ascontiguousarray(ms[1], dtype=np.float64)
            return MeshSetView(len(off) - 1, ptr(off, PU64), ptr(tris)), (off, tris)
        rv, keep_r = view(R)
        sv, keep_s = view(S) if S is not None else (None, None)
        res = ExhaustiveResult()
        self.check(self.lib.tj_exhaustive_join(self.ctx, ctypes.byref(rv), ctypes.byref(sv) if sv else None,
                                               ctypes.c_int32(self.TYPES[type]), ctypes.c_double(tau),
                                               ctypes.c_uint32(k), ctypes.byref(res)))
        out = [(res.r[i], res.s[i], res.d[i], res.rank[i]) for i in range(res.n_records)]
        self.lib.tj_exhaustive_result_free(ctypes.byref(res))
        return out

    def refine_batch(self, tris, hd, ph, r_off, s_off, r_len, s_len, flags=0):
        n = len(r_off)
        lb = np.zeros(n)
        ub = np.zeros(n)
        tris = np.ascontiguousarray(tris, dtype=np.float64)
        hd = np.ascontiguousarray(hd, dtype=np.float64)
        ph = np.ascontiguousarray(ph, dtype=np.float64)
        r_off = np.ascontiguousarray(r_off, dtype=np.uint64)
        s_off = np.ascontiguousarray(s_off, dtype=np.uint64)
        r_len = np.ascontiguousarray(r_len, dtype=np.uint32)
        s_len = np.ascontiguousarray(s_len, dtype=np.uint32)
        self.check(self.lib.tj_refine_batch(self.ctx, ctypes.c_uint64(len(hd)), ptr(tris), ptr(hd), ptr(ph),
                                            ctypes.c_uint64(n), ptr(r_off, PU64), ptr(s_off, PU64),
                                            ptr(r_len, PU32), ptr(s_len, PU32), ctypes.c_uint32(flags),
                                            ptr(lb), ptr(ub)))
        return lb, ub

    def load(self, path):
        h = ctypes.c_void_p()
        rc = self.lib.tj_host_dataset_load(path.encode(), ctypes.byref(h))
        if rc != 0:
            raise RuntimeError(f"tj_host_dataset_load({path}) = {rc}")
        ds = ctypes.c_void_p()
        try:
            self.check(self.lib.tj_dataset_upload(self.ctx, self.lib.tj_host_dataset_view(h), ctypes.byref(ds)))
        finally:
            self.lib.tj_host_dataset_free(h)
        return ds

    def join(self, R, S, type="within", tau=0.0, k=1, lods=(20, 40, 60, 80, 100), flags=0, refine_chunk=500000,
             shard=(0, 1), exact=False):
        arr = (ctypes.c_uint32 * len(lods))(*lods)
        if exact:
            flags |= 8  # TJ_FLAG_EXACT_RECOMPUTE
        spec = JoinSpec(self.TYPES[type], tau, k, 4194304, refine_chunk, len(lods), arr, 1, flags, shard[0],
                        shard[1], 1024)
        res = JoinResult()
        rc = self.lib.tj_join(self.ctx, R, S, ctypes.byref(spec), None, ctypes.byref(res))
        if rc != 0:
            msg = self.err()
            raise RuntimeError(f"tj_join status {rc}: {msg}")
        n = res.n_cands
        out = {
            "pair_r": np.ctypeslib.as_array(res.pair_r, (max(n, 1),))[:n].copy(),
            "pair_s": np.ctypeslib.as_array(res.pair_s, (max(n, 1),))[:n].copy(),
            "lb": np.ctypeslib.as_array(res.lb, (max(n, 1),))[:n].copy(),
            "ub": np.ctypeslib.as_array(res.ub, (max(n, 1),))[:n].copy(),
            "status": np.ctypeslib.as_array(res.status, (max(n, 1),))[:n].copy(),
            "decided_at": np.ctypeslib.as_array(res.decided_at, (max(n, 1),))[:n].copy(),
            "nq": res.n_queries, "vp_generated": res.vp_generated, "vp_pruned": res.vp_pruned,
            "levels": [(res.level[i], res.level_vps[i], res.level_facet_pairs[i]) for i in range(res.n_levels_run)],
            "decision_mode": res.decision_mode,
            "queue_reruns": res.queue_reruns,
            "mat_chunks": res.mat_chunks,
        }
        self.lib.tj_join_result_free(ctypes.byref(res))
        return out

    def free(self, ds):
        self.lib.tj_dataset_free(ds)


def records_from_candidates(c, knn):
    """Reference record assembly (proj/src/engine.cpp:161-185) over tj_join result arrays."""
    recs = []
    conf = np.nonzero(c["status"] == 1)[0]
    if not knn:
        for op in conf:
            recs.append((int(c["pair_r"][op]), int(c["pair_s"][op]), float(c["lb"][op]), float(c["ub"][op]),
                         stage_name(int(c["decided_at"][op])), 0))
        return recs
    by_r = {}
    for op in conf:
        by_r.setdefault(int(c["pair_r"][op]), []).append(op)
    for r in sorted(by_r):
        ops = sorted(by_r[r], key=lambda o: (c["ub"][o], c["lb"][o], c["pair_s"][o]))
        for rank, op in enumerate(ops, 1):
            recs.append((r, int(c["pair_s"][op]), float(c["lb"][op]), float(c["ub"][op]),
                         stage_name(int(c["decided_at"][op])), rank))
    return recs


# ---------------------------------------------------------------- C restatement oracle
class OraRecord(ctypes.Structure):
    _fields_ = [("r", ctypes.c_uint32), ("s", ctypes.c_uint32), ("lb", ctypes.c_double), ("ub", ctypes.c_double),
                ("stage", ctypes.c_int16), ("rank", ctypes.c_uint32)]


class OraStage(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int16)] + [(n, ctypes.c_uint64) for n in
                                             ["pairs_in", "confirmed", "removed", "pairs_out", "vp_generated",
                                              "vp_pruned", "facet_pairs"]]


class OraResult(ctypes.Structure):
    _fields_ = [("n_records", ctypes.c_uint64), ("records", ctypes.POINTER(OraRecord)), ("n_stages", ctypes.c_uint32),
                ("stages", OraStage * 20), ("error", ctypes.c_char * 256), ("status", ctypes.c_int)]


def load_oracle():
    return ctypes.CDLL(ORACLE_LIB)


def oracle_join(lib, r_path, s_path, type="within", tau=0.0, k=1, lods=(20, 40, 60, 80, 100), exact=False):
    res = OraResult()
    arr = (ctypes.c_uint32 * len(lods))(*lods)
    lib.ora_join_files_ex(r_path.encode(), (s_path or "").encode(), Capi.TYPES[type], ctypes.c_double(tau), k, arr,
                          len(lods), 1 if exact else 0, ctypes.byref(res))
    if res.status != 0:
        raise RuntimeError(res.error.decode())
    recs = [(x.r, x.s, x.lb, x.ub, stage_name(x.stage), x.rank) for x in res.records[:res.n_records]]
    stages = [{"stage": stage_name(x.code), "pairs_in": x.pairs_in, "confirmed": x.confirmed, "removed": x.removed,
               "pairs_out": x.pairs_out, "vp_generated": x.vp_generated, "vp_pruned": x.vp_pruned,
               "facet_pairs": x.facet_pairs} for x in res.stages[:res.n_stages]]
    lib.ora_result_free(ctypes.byref(res))
    return recs, stages


# ---------------------------------------------------------------- golden fixtures
def golden(name):
    return os.path.join(GOLDEN, name)


def golden_joins(name="joins.json"):
    with open(golden(name)) as f:
        joins = json.load(f)
    for j in joins:
        j["records"] = [tuple(r) for r in j["records"]]
    return joins


def adversarial_joins():
    """tests/golden/adversarial_joins.json (tests/golden/make_adversarial.py, the reference)."""
    return golden_joins("adversarial_joins.json")


def join_id(j):
    kw = ",".join(f"{k}={v}" for k, v in sorted(j["kwargs"].items()) if k != "lods")
    return f"{j['r']}-{j['s'] or 'self'}-{kw}"


def load_staged(path):
    """Parse an oracle/ref_shim.cpp ref_staged_dump file."""
    with open(path, "rb") as f:
        data = f.read()
    pos = 0
    (nc,) = struct.unpack_from("<Q", data, pos)
    pos += 8
    cand_dt = np.dtype([("r", "<u4"), ("s", "<u4"), ("lb", "<f8"), ("ub", "<f8"), ("st", "u1"), ("at", "<i2")])
    cands = np.frombuffer(data, dtype=cand_dt, count=nc, offset=pos)
    pos += nc * cand_dt.itemsize
    (na,) = struct.unpack_from("<Q", data, pos)
    pos += 8
    active = np.frombuffer(data, dtype=np.uint32, count=3 * na, offset=pos).reshape(na, 3)
    pos += 12 * na
    (nl,) = struct.unpack_from("<I", data, pos)
    pos += 4
    levels = []
    for _ in range(nl):
        level, fp = struct.unpack_from("<IQ", data, pos)
        pos += 12
        lb = np.frombuffer(data, dtype=np.float64, count=na, offset=pos)
        pos += 8 * na
        ub = np.frombuffer(data, dtype=np.float64, count=na, offset=pos)
        pos += 8 * na
        levels.append((level, fp, lb, ub))
    return cands, active, levels


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)
