"""Multi-GPU plumbing for one-process-per-GPU launches (torchrun).

The join shards by query object: query r belongs to shard ``(r // block) % n_shards``
(blocks of ``block`` consecutive queries dealt round-robin, so dense and sparse regions
spread over the GPUs). Every shard runs the whole pipeline for its queries against all of
S with no communication (``TRIJOIN_PROCESS_SHARD=i/n`` makes ``run_join`` join shard i only,
``csrc/host/engine.cpp``). The only exchange is at the end of a join:

  * ``gather_records``: the records of every rank to rank 0 — an all-gather of the record
    counts (one int64 per rank), then the 32-byte records themselves, padded to the largest
    rank's count (NCCL has no gather-v), over NCCL / NVLink when the tensors live on the GPU.
    Records are grouped by query and each query lives on exactly one rank, so a stable sort
    by r reproduces the single-process record order (reference ``src/engine.cpp:161-185``).
  * ``merge_stats``: the stage counters of every rank summed (wall times: max), which equals
    the single-process join's counters because each rank counts its own queries' pairs.
"""
import json

import numpy as np

BLOCK = 1024

# The record layout of ``_core.join_datasets(..., records="array")``.
REC_DTYPE = np.dtype({"names": ["r", "s", "lb", "ub", "stage", "rank"],
                      "formats": ["<u4", "<u4", "<f8", "<f8", "<i2", "<u4"],
                      "offsets": [0, 4, 8, 16, 24, 28], "itemsize": 32})

_COUNTERS = ("pairs_in", "confirmed", "removed", "pairs_out", "vp_generated", "vp_pruned", "facet_pairs")


def shard_of(r, n_shards, block=BLOCK):
    """Shard owning query r (the partition run_join and Resident use)."""
    return (np.asarray(r, dtype=np.int64) // block) % n_shards


def shard_queries(n_queries, index, count, block=BLOCK):
    """Ascending query ids of shard ``index`` of ``count``."""
    r = np.arange(n_queries, dtype=np.int64)
    return r[shard_of(r, count, block) == index]


def gather_records(recs, dst=0, group=None, device=None):
    """Every rank's records (``REC_DTYPE`` array of its own queries) to rank ``dst``, merged into
    the single-process order; other ranks get None. ``device``: where the exchange tensors live
    (a CUDA device for NCCL, None = CPU for gloo)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    recs = np.ascontiguousarray(recs)
    if recs.dtype != REC_DTYPE:  # same 32-byte layout under another dtype object (pybind11-made)
        if recs.dtype.itemsize != REC_DTYPE.itemsize:
            raise ValueError(f"records must be {REC_DTYPE}, got {recs.dtype}")
        recs = recs.view(np.uint8).view(REC_DTYPE)
    dev = torch.device("cpu") if device is None else torch.device(device)
    n = torch.tensor([len(recs)], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    width = max(1, max(counts)) * REC_DTYPE.itemsize
    buf = torch.zeros(width, dtype=torch.uint8, device=dev)
    if len(recs):
        buf[:recs.nbytes] = torch.from_numpy(recs.view(np.uint8)).to(dev, non_blocking=False)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    if rank != dst:
        return None
    merged = np.concatenate([parts[i][:counts[i] * REC_DTYPE.itemsize].cpu().numpy().view(REC_DTYPE)
                             for i in range(world)])
    return merged[np.argsort(merged["r"], kind="stable")]


def merge_stats(stats):
    """Stats dicts (or JSON strings) of every rank's shard -> the whole join's stats."""
    stats = [json.loads(s) if isinstance(s, str) else s for s in stats]
    out = json.loads(json.dumps(stats[0]))
    out["results"] = sum(s["results"] for s in stats)
    out["total_ms"] = max(s["total_ms"] for s in stats)
    for i, st in enumerate(out["stages"]):
        for key in _COUNTERS:
            if key in st:
                st[key] = sum(s["stages"][i][key] for s in stats)
        st["wall_ms"] = max(s["stages"][i]["wall_ms"] for s in stats)
    return out


def gather_stats(stats_json, dst=0, group=None):
    """merge_stats over every rank's stats JSON, on rank ``dst`` (None elsewhere)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    got = [None] * world
    dist.all_gather_object(got, stats_json, group=group)
    return merge_stats(got) if dist.get_rank(group) == dst else None


def records_to_tuples(arr):
    """REC_DTYPE array -> the reference's record tuples (r, s, lb, ub, stage name, rank)."""
    names = {-3: "undecided", -2: "mbb", -1: "voxel", 100: "exact"}
    return [(int(x["r"]), int(x["s"]), float(x["lb"]), float(x["ub"]),
             names.get(int(x["stage"]), f"lod-{int(x['stage'])}"), int(x["rank"])) for x in arr]
