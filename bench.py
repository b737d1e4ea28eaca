#!/usr/bin/env python3
"""Benchmark: candidate object-pairs refined/sec of the B200 trijoin engine (BASELINE.json).

A *step* is one full filter-and-refine join (MBB filter -> voxel-pair filter -> LOD 20/60/100
refinement) of configuration B by default: intersection join of 100k x 100k synthetic nuclei
(312-facet spheres) on one B200 (BASELINE.json configs[1]). Metric units are the candidate
object pairs entering the voxel + LOD cascade (stats stages["voxel"].pairs_in).

  value : device-resident datasets (uploaded once), K timed joins; CUDA events on the host
          stream bracketing each blocking tj_join call, barrier + synchronize around the loop,
          max over ranks.
  e2e   : the public API with host buffers (`join_datasets`: pack -> H2D -> join -> D2H ->
          records), same metric.
  roofline: the dominant kernel k_screen (CUDA events around its launches on its stream):
          FLOPs = box tests x 20 (counted on the device) vs the FP32 peak
          148 SM x 128 lanes x 2 x sm_max_mhz (MEASURED_PEAKS.json); its largest launch alone,
          and all refinement kernels (+ evaluated facet pairs x 1500) beside it. traffic: DRAM
          bytes of one k_screen launch from the committed ncu --set full capture.
  cpu_baseline: the reference's own run_join (oracle/_ref, built from /root/reference) on a
          deterministic R-slice of the same workload on all host cores (rank 0, N=1 only).

--impl reference runs only the reference CPU arm (rank 0; other ranks exit 0).
Multi-GPU (torchrun): query objects are sharded in blocks of 1024 across ranks (no data-path
collective); each rank uploads only its own queries. In the e2e run every step ends with the
records of all ranks gathered to rank 0 over NCCL (paper_2604_19982_b200.dist.gather_records:
counts all-gather + padded record all-gather, stable merge by query), inside the timed region.
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# roofline.achieved follows SURVEY §8(d): 1,500 FLOP per exact facet-pair evaluation + 20 FLOP per
# culling box test, counted on the device. The builder's finer model (25 per box test, 300 per
# separating-axis test) is reported beside it as roofline.builder_model.
FLOP_PER_PAIR = 1500.0   # exact FP64 evaluation: dynamic op count of tri_tri_distance + padding
FLOP_PER_TEST = 20.0     # culling box test
B_FLOP_PER_TEST = 25.0   # builder model: stage-1 FP32 test (facet-AABB gap + thresholds)
B_FLOP_PER_SAT = 300.0   # builder model: stage-2 FP32 separating-axis bound (2 face + 9 edge axes)
TYPE_CODE = {"within": 0, "intersect": 1, "knn": 2}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="B")
    p.add_argument("--scale", type=float, default=1.0, help="object-count scale (same density)")
    p.add_argument("--data-dir", default=os.environ.get("TRIJOIN_BENCH_DIR", "/tmp/trijoin_bench"))
    p.add_argument("--cpu-stride", type=int, default=100, help="R-slice stride of the CPU baseline sample")
    p.add_argument("--ref-stride", type=int, default=250, help="R-slice stride per --impl reference step")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cull", action="store_true", help="disable exact-preserving culling (A/B)")
    p.add_argument("--profile", action="store_true", help="one resident join only (for ncu)")
    p.add_argument("--residency", default="auto", choices=["auto", "compact", "expanded"],
                   help="device residency of the value-leg datasets (auto: compact for D, E)")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def ncu_traffic(config):
    """DRAM bytes of one k_screen launch (the dominant kernel) from the committed ncu --set full
    capture of this workload (profiles/ncu_traffic_<config>.json, scripts/ncu_traffic.py), or None."""
    path = os.path.join(ROOT, "profiles", f"ncu_traffic_{config}.json")
    try:
        launches = [l for l in json.load(open(path))["launches"] if l["kernel"] == "k_screen"]
    except (OSError, ValueError, KeyError):
        return None, None
    if not launches:
        return None, None
    top = max(launches, key=lambda l: l["dram_bytes"])
    return top["dram_bytes"], f"profiles/ncu_traffic_{config}.json ({top['report']}: one k_screen launch, " \
                              f"{top['duration_s'] * 1e3:.2f} ms, {top['dram_GBps']:.0f} GB/s)"


def ncu_pipes(config):
    """ncu pipe utilisation of the dominant refinement launch from the committed --set full
    capture (profiles/ncu_pipes_<config>.json, scripts/ncu_table.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", f"ncu_pipes_{config}.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"sm_max_mhz": 1965.0, "hbm_gbs": 6650.0}, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, path, gpu):
        self.path, self.proc = path, None
        if os.environ.get("BENCH_NO_CLOCKS"):
            return
        try:
            self.f = open(path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu), "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = float(parts[2])
                except ValueError:
                    continue
                for n, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def ref_shim():
    lib = ctypes.CDLL(os.path.join(ROOT, "oracle", "_ref", "libref_shim.so"))
    lib.ref_join_timed_records.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_double,
                                           ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32), ctypes.c_uint32,
                                           ctypes.c_uint, ctypes.c_uint32, ctypes.POINTER(ctypes.c_double),
                                           ctypes.c_char_p]
    lib.ref_last_error.restype = ctypes.c_char_p
    return lib


REC_DTYPE = np.dtype([("r", "<u4"), ("s", "<u4"), ("lb", "<f8"), ("ub", "<f8"), ("stage", "<i2"), ("pad", "<i2"),
                      ("rank", "<u4")])


def stage_name(code):
    """Reference stage_name (proj/src/engine.cpp: mbb / voxel / lod-L, 100 -> exact)."""
    code = int(code)
    return {-3: "undecided", -2: "mbb", -1: "voxel", 100: "exact"}.get(code, f"lod-{code}")


def ref_join(lib, r_path, s_path, kw, lods, workers, repeats=1, records_path=None):
    """The reference's own run_join on the host cores; loads untimed, joins timed. With
    `records_path` the last join's records are returned as (r, s, lb, ub, stage, rank) tuples."""
    arr = (ctypes.c_uint32 * len(lods))(*lods)
    out = (ctypes.c_double * 6)()
    rc = lib.ref_join_timed_records(r_path.encode(), s_path.encode(), TYPE_CODE[kw["type"]],
                                    float(kw.get("tau", 0.0)), int(kw.get("k", 1)), arr, len(lods), workers, repeats,
                                    out, records_path.encode() if records_path else None)
    if rc != 0:
        raise RuntimeError("reference join failed: " + lib.ref_last_error().decode())
    res = {"ms": out[0], "pairs_in": out[1], "facet_pairs": out[2], "results": out[3], "cores": int(out[4])}
    if records_path:
        rec = np.fromfile(records_path, dtype=REC_DTYPE)
        res["records"] = [(int(x["r"]), int(x["s"]), float(x["lb"]), float(x["ub"]), stage_name(x["stage"]),
                           int(x["rank"])) for x in rec]
    return res


def slice_parity(gpu_records, ref_records, stride, s_ids=None):
    """Bitwise comparison of the GPU's records of queries r % stride == 0 with the reference's
    records of the R-slice (slice query r' is query r' * stride; per-query independence,
    SURVEY §8e; with s_ids the slice's S file holds only those S objects: s' -> s_ids[s']).
    lb / ub compare as IEEE bit patterns."""
    def key(rec):
        r, s, lb, ub, stage, rank = rec
        return (r, s, np.float64(lb).view(np.uint64).item(), np.float64(ub).view(np.uint64).item(), stage, rank)
    mine = [key(x) for x in gpu_records if x[0] % stride == 0]
    theirs = [key((r * stride, int(s_ids[s]) if s_ids is not None else s) + tuple(rest))
              for r, s, *rest in ref_records]
    mismatches = sum(1 for a, b in zip(mine, theirs) if a != b) + abs(len(mine) - len(theirs))
    return {"stride": stride, "slice_records": len(theirs), "gpu_records": len(mine), "mismatches": mismatches,
            "compared": "r, s, lb bits, ub bits, stage, rank of every record, in the reference's order"}


def load_synth_tables():
    """paper_2604_19982_b200/synth.py loaded as a plain module (its CONFIGS / LODS tables)
    without importing the package, so the reference arm never maps this repo's libraries."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("tj_synth_tables",
                                                  os.path.join(ROOT, "paper_2604_19982_b200", "synth.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


# Configurations built in memory (their full index files would not fit the box's disk): the
# reference's R-slice runs against only the S objects near the slice (synth.write_slice_files).
IN_MEMORY = ("D", "E")


def build_slice_subprocess(name, data_dir, scale, stride):
    """Slice index files for the reference arm, written by a separate process so the timed
    reference process maps only oracle/_ref (the writer is this repo's replicate_index)."""
    if name in IN_MEMORY:
        code = ("import sys, json; sys.path.insert(0, %r); from paper_2604_19982_b200 import synth; "
                "r, s, ri, si = synth.write_slice_files(%r, %r, %d, %r); print(json.dumps([r, s]))"
                % (ROOT, name, scale, stride, data_dir))
    else:
        code = ("import sys, json; sys.path.insert(0, %r); from paper_2604_19982_b200 import synth; "
                "print(json.dumps(synth.build_config(%r, %r, scale=%r, r_stride=%d)))" % (ROOT, name, data_dir, scale,
                                                                                         stride))
    out = subprocess.run([sys.executable, "-c", code], check=True, capture_output=True, text=True).stdout
    return tuple(json.loads(out.strip().splitlines()[-1]))


def main():
    a = parse()
    world, rank, local = dist_env()
    synth = load_synth_tables()

    name = a.config
    _, _, kw = synth.CONFIGS[name]
    lods = list(synth.LODS)
    workload = {
        "A": "A: within-tau 0.5, 1k nuclei (1012 f) x 1k vessels (1012 f)",
        "B": "B: intersection join, 100k x 100k nuclei (312-facet spheres)",
        "C": "C: k-NN k=3, 200k nuclei x 10k vessels",
        "D": "D: within-tau 0.2, 1M x 1M nuclei",
        "E": "E: within-tau 0, 50k scanned-surface meshes (~20k facets) self-join",
    }[name]
    data_dir = os.path.join(a.data_dir, f"{name}_x{a.scale:g}")

    if a.impl == "reference":
        if rank != 0:
            return 0
        r_slice, s_path = build_slice_subprocess(name, data_dir, a.scale, a.ref_stride)
        lib = ref_shim()
        workers = os.cpu_count() or 1
        times, last = [], None
        for i in range(a.warmup + a.steps):
            last = ref_join(lib, r_slice, s_path, kw, lods, workers)
            if i >= a.warmup:
                times.append(last["ms"])
        ms = float(np.mean(times))
        value = last["pairs_in"] / (ms / 1e3)
        sample = (f"R-slice every {a.ref_stride}th query object of {workload} vs the full S "
                  f"({int(last['pairs_in'])} candidate pairs, {int(last['facet_pairs'])} facet pairs per step)")
        line = {"metric": "candidate object-pairs refined/sec", "value": value, "unit": "pairs/s",
                "impl": "reference", "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": {"workload": workload, "lods": lods, "sample": sample},
                "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": last["cores"], "kind": "reference",
                                 "sample": sample},
                "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import torch.distributed as dist

    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        os.environ["TRIJOIN_PROCESS_SHARD"] = f"{rank}/{world}"  # e2e: this rank's query blocks
    os.environ.setdefault("TRIJOIN_DEVICES", str(local))
    import paper_2604_19982_b200 as tj
    from paper_2604_19982_b200 import _core
    from paper_2604_19982_b200 import dist as tjdist
    from paper_2604_19982_b200 import synth

    # ---- inputs (built once per box; node-local rank 0 writes, others wait) ----
    t_setup = time.time()
    in_memory = name in IN_MEMORY
    if in_memory:  # translated template copies straight into memory (no index files)
        R, S, _ = synth.build_datasets(name, scale=a.scale)
    else:
        if local == 0:
            r_path, s_path = synth.build_config(name, data_dir, scale=a.scale)
        if world > 1:
            dist.barrier()
        r_path, s_path = synth.build_config(name, data_dir, scale=a.scale)
        R = tj.load_dataset(r_path)
        S = tj.load_dataset(s_path) if s_path else R  # "" = self-join (config E)
    # each rank uploads only its own query shard of R (blocks of 1024 queries dealt round-robin);
    # D / E: the expanded form exceeds HBM, so the datasets stay compact-resident and each
    # level's active voxels are expanded on demand (TJ_DATASET_COMPACT)
    compact = a.residency == "compact" or (a.residency == "auto" and in_memory)
    res = tj.Resident(R, S, device=local, shard_index=rank, shard_count=world, compact=compact)
    setup_s = time.time() - t_setup
    flags = 1 if a.no_cull else 0
    run_kw = dict(type=kw["type"], tau=float(kw.get("tau", 0.0)), k=int(kw.get("k", 1)), lods=lods, flags=flags)

    if a.profile:
        out = res.run(**run_kw)
        if rank == 0:
            print(json.dumps({"profile": True, "total_ms": out["total_ms"], "levels": out["levels"]}))
        return 0

    dev = torch.device("cuda", local)
    # the clocks sampler starts before the warm-up (its first NVML queries must not land in
    # the timed region); it keeps sampling through the timed steps
    clocks = Clocks(os.path.join(ROOT, "gpurun_out", f"clocks_rank{rank}.csv") if os.path.isdir(
        os.path.join(ROOT, "gpurun_out")) else f"/tmp/trijoin_clocks_{rank}.csv", local)
    for _ in range(a.warmup):
        res.run(**run_kw)
    launches0 = _core.kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
    evs[0].record()
    outs = []
    for i in range(a.steps):
        outs.append(res.run(**run_kw))
        evs[i + 1].record()
    torch.cuda.synchronize(dev)
    e0, e1 = evs[0], evs[-1]
    step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(a.steps)]
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = _core.kernel_launches() - launches0
    elapsed_ms = e0.elapsed_time(e1)
    pairs = float(outs[-1]["voxel_pairs_in"])
    fp = float(sum(l["facet_pairs"] for l in outs[-1]["levels"]))
    evaluated = float(sum(l["evaluated"] for l in outs[-1]["levels"]))
    tested = float(sum(l["tested"] for l in outs[-1]["levels"]))
    screened = float(sum(l["screened"] for l in outs[-1]["levels"]))
    kernel_ms = float(np.mean([sum(l["kernel_ms"] for l in o["levels"]) for o in outs]))
    # the dominant kernel (k_screen): its launches' CUDA-event time, and its largest launch (the
    # last level's) alone
    screen_ms = float(np.mean([sum(l.get("screen_ms", 0.0) for l in o["levels"]) for o in outs]))
    top_lv = max(outs[-1]["levels"], key=lambda l: l.get("screen_ms", 0.0))
    top_ms = float(np.mean([[l for l in o["levels"] if l["level"] == top_lv["level"]][0].get("screen_ms", 0.0)
                            for o in outs]))
    top_tested = float(top_lv["tested"])
    stats = torch.tensor([elapsed_ms, pairs, fp, evaluated, tested, kernel_ms, screened, screen_ms, top_ms,
                          top_tested], dtype=torch.float64, device=dev)
    if world > 1:
        mx = stats.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = stats.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        elapsed_ms, kernel_ms = float(mx[0]), float(mx[5])
        pairs, fp, evaluated, tested = (float(sm[i]) for i in range(1, 5))
        screened = float(sm[6])
        screen_ms, top_ms, top_tested = float(mx[7]), float(mx[8]), float(sm[9])
    ms_per_step = elapsed_ms / a.steps
    value = pairs / (ms_per_step / 1e3)

    peaks, peak_src = measured_peaks()
    fp32_peak = 148 * 128 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12  # TFLOP/s
    work_flop = evaluated * FLOP_PER_PAIR + tested * FLOP_PER_TEST
    achieved = work_flop / (kernel_ms / 1e3) / 1e12 / max(world, 1)
    b_flop = evaluated * FLOP_PER_PAIR + tested * B_FLOP_PER_TEST + screened * B_FLOP_PER_SAT
    b_achieved = b_flop / (kernel_ms / 1e3) / 1e12 / max(world, 1)
    brute_peak_pairs = fp32_peak * 1e12 / FLOP_PER_PAIR  # every reference facet pair through tri_tri at FP32 peak
    traffic, traffic_src = ncu_traffic(a.config)
    # SURVEY 8(d) for the dominant kernel k_screen: 20 FLOP per box test it runs (counted on the
    # device) / its launches' CUDA-event time (the exact FP64 evaluations are k_eval's work)
    s_achieved = tested * FLOP_PER_TEST / (screen_ms / 1e3) / 1e12 / max(world, 1) if screen_ms else None
    t_achieved = top_tested * FLOP_PER_TEST / (top_ms / 1e3) / 1e12 / max(world, 1) if top_ms else None
    roofline = {"bound": "fp32", "achieved": s_achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                "frac": s_achieved / fp32_peak if s_achieved else None, "traffic": traffic,
                "traffic_source": traffic_src,
                "kernel": f"k_screen (the dominant kernel: {screen_ms:.1f} of {elapsed_ms / a.steps:.1f} ms per join; "
                          "all its launches in the timed region, CUDA events on its stream)",
                "flop_model": f"SURVEY 8(d): {FLOP_PER_TEST:g} FLOP per box test (counted on the device)",
                "largest_launch": {"level": top_lv["level"], "ms": top_ms, "box_tests": top_tested,
                                   "achieved": t_achieved, "frac": t_achieved / fp32_peak if t_achieved else None},
                "all_refinement": {"kernels": "k_seed + k_screen + k_eval, all levels", "achieved": achieved,
                                   "frac": achieved / fp32_peak, "kernel_ms": kernel_ms,
                                   "flop_model": f"{FLOP_PER_PAIR:g} x exact FP64 evaluations + {FLOP_PER_TEST:g} x "
                                                 "box tests"},
                "builder_model": {"achieved": b_achieved, "frac": b_achieved / fp32_peak,
                                  "flop_model": f"{B_FLOP_PER_TEST:g} x box tests + {B_FLOP_PER_SAT:g} x "
                                                f"separating-axis tests + {FLOP_PER_PAIR:g} x exact evaluations"},
                "ncu_pipes": ncu_pipes(a.config),
                "peak_source": f"148 SM x 128 FP32 lanes x 2 x sm_max_mhz ({peak_src} MEASURED_PEAKS.json)",
                "pairs_evaluated_per_s": evaluated / (kernel_ms / 1e3) / max(world, 1),
                "ref_equiv_facet_pairs_per_s": fp / (kernel_ms / 1e3) / max(world, 1),
                "ref_equiv_vs_brute_force_peak": fp / (kernel_ms / 1e3) / max(world, 1) / brute_peak_pairs,
                "cull_skip_frac": 1.0 - evaluated / fp if fp else None}

    # ---- e2e: public API from host buffers ----
    # the e2e leg uploads its own copies: release the resident datasets first (their pooled
    # device memory is reused)
    res_bytes, n_q = res.device_bytes, res.n_queries
    del res
    e2e = None
    gpu_records = None
    if not a.no_e2e:
        ts = []
        parts = []
        d2h = 0
        for i in range(max(1, min(a.steps, 3)) + 1):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            recs, js = _core.join_datasets(R, S, type=kw["type"], tau=float(kw.get("tau", 0.0)),
                                           k=int(kw.get("k", 1)), lods=lods, records="array")
            if world > 1:  # records of every rank's shard to rank 0 (NCCL), merged in query order
                recs = tjdist.gather_records(recs, device=dev)
            torch.cuda.synchronize(dev)
            t1 = time.perf_counter()
            if i > 0:
                ts.append((t1 - t0) * 1e3)
            gpu_records = recs
            st = json.loads(js)
            n_c = st["stages"][0]["pairs_in"] - st["stages"][0]["removed"]
            d2h = n_c * (4 + 4 + 8 + 8 + 1 + 2) + (n_q + 1) * 8 + n_q * 4
            pairs_e2e = st["stages"][1]["pairs_in"]
            if i > 0:
                b = dict(st.get("b200", {}))
                b["run_join_ms"] = st.get("total_ms", 0.0)
                b["python_ms"] = (t1 - t0) * 1e3 - b["run_join_ms"]
                parts.append(b)
            h2d = st.get("b200", {}).get("h2d_bytes", 0)
        e2e_ms = float(np.mean(ts))
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        tot = torch.tensor([float(pairs_e2e), float(h2d), float(d2h)], dtype=torch.float64, device=dev)
        if world > 1:  # each rank joined its own query blocks (TRIJOIN_PROCESS_SHARD)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        pairs_e2e, h2d, d2h = float(tot[0]), float(tot[1]), float(tot[2])
        e2e = {"value": pairs_e2e / (float(t[0]) / 1e3), "unit": "pairs/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": float(t[0]),
               "path": "paper_2604_19982_b200._core.join_datasets -> trijoin::run_join -> tj_join (C-ABI)",
               "breakdown_ms": {k: round(float(np.mean([p.get(k, 0.0) for p in parts])), 2)
                                for k in ("pack_ms", "upload_ms", "device_ms", "stream_wait_ms", "run_join_ms",
                                          "python_ms")},
               "steps_ms": [round(x, 1) for x in ts],
               "timeline_ms": parts[-1].get("timeline", {}) if parts else {}}

    cpu = None
    parity = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            s_ids = None
            if in_memory:
                r_slice, s_full, _, s_ids = synth.write_slice_files(name, a.scale, a.cpu_stride, data_dir + "_slice")
            else:
                r_slice, s_full = synth.build_config(name, data_dir + "_slice", scale=a.scale, r_stride=a.cpu_stride)
            if gpu_records is None:  # the public API's records of the full workload (untimed)
                gpu_records, _ = _core.join_datasets(R, S, type=kw["type"], tau=float(kw.get("tau", 0.0)),
                                                     k=int(kw.get("k", 1)), lods=lods, records="array")
            gpu_records = tjdist.records_to_tuples(gpu_records)
            rec_path = os.path.join(data_dir + "_slice", "ref_records.bin")
            rj = ref_join(ref_shim(), r_slice, s_full, kw, lods, os.cpu_count() or 1, records_path=rec_path)
            parity = slice_parity(gpu_records, rj["records"], a.cpu_stride, s_ids)
            parity["slice_candidates"] = int(rj["pairs_in"])
            cpu = {"value": rj["pairs_in"] / (rj["ms"] / 1e3), "unit": "pairs/s", "cores": rj["cores"],
                   "kind": "reference",
                   "sample": f"reference run_join (oracle/_ref) on every {a.cpu_stride}th query object vs "
                             f"{('the ' + str(len(s_ids)) + ' S objects near the slice') if in_memory else 'the full S'}: "
                             f"{int(rj['pairs_in'])} candidate pairs, {int(rj['facet_pairs'])} facet pairs, "
                             f"{rj['ms'] / 1e3:.1f} s",
                   "facet_pairs_per_s": rj["facet_pairs"] / (rj["ms"] / 1e3)}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "pairs/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {"metric": "candidate object-pairs refined/sec", "value": value, "unit": "pairs/s", "n_gpus": world,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (replicated preprocessed sphere templates, reference generator placement)",
                "config": {"workload": workload, "lods": lods, "scale": a.scale,
                           "candidate_pairs": pairs, "facet_pairs_ref_count": fp,
                           "join_wall_ms": ms_per_step, "l2": "inputs larger than L2 "
                           f"({res_bytes / 1e9:.1f} GB resident)", "parallelism": f"r-shard x{world}",
                           "setup_s": round(setup_s, 1), "cull": not a.no_cull,
                           "step_ms": [round(x, 2) for x in step_ms],
                           "filter_last_step": {k: outs[-1][k] for k in ("n_cands", "voxel_pairs_in", "vp_generated",
                                                                      "vp_pruned", "confirmed", "mbb_ms",
                                                                      "voxel_ms")},
                           "levels_last_step": outs[-1]["levels"]},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
                "gpu_launches": int(launches), "parity": parity}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    if parity is not None and parity["mismatches"]:
        print(f"PARITY FAILURE: {parity['mismatches']} record mismatches against the reference slice",
              file=sys.stderr)
        return 3
    return 0


if __name__ == "__main__":
    sys.exit(main())
