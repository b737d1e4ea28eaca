"""Multi-rank host logic on CPU (gloo, world_size 2) through the product's own plumbing
(paper_2604_19982_b200/dist.py): the query-shard partition run_join uses, the end-of-join
record gather (counts all-gather + padded record all-gather, stable merge by query) and the
stage-counter merge. The records are synthetic (no GPU here); tests/test_gpu_multiproc.py
runs the same path on real joins."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_19982_b200 import dist as tjdist


def _records(nq, seed, knn=False):
    rng = np.random.default_rng(seed)
    rows = []
    for r in range(nq):
        k = int(rng.integers(0, 4))
        for i, s in enumerate(sorted(rng.choice(5000, size=k, replace=False))):
            rows.append((r, int(s), float(rng.random()), float(rng.random() + 1), 60, i + 1 if knn else 0))
    out = np.zeros(len(rows), dtype=tjdist.REC_DTYPE)
    for i, row in enumerate(rows):
        out[i] = row
    return out


def _worker(rank, world, port, nq, block, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = _records(nq, 5, knn=True)
    mine = full[np.isin(full["r"], tjdist.shard_queries(nq, rank, world, block))]  # this rank's shard
    merged = tjdist.gather_records(mine)
    stats = {"results": len(mine), "total_ms": 1.0 + rank,
             "stages": [{"name": "mbb", "wall_ms": 1.0 + rank, "pairs_in": 100 * (rank + 1), "confirmed": rank,
                         "removed": 7, "pairs_out": 3}]}
    st = tjdist.gather_stats(stats)
    if rank == 0:
        ok = len(merged) == len(full) and bool((merged == full).all())
        ok = ok and st["results"] == len(full) and st["stages"][0]["pairs_in"] == 300 and \
            st["stages"][0]["confirmed"] == 1 and st["stages"][0]["wall_ms"] == 2.0
        out.put(ok)
    else:
        assert merged is None and st is None
    dist.destroy_process_group()


def _run(nq, block):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, nq, block, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    return ok


def test_gather_reproduces_single_rank_order():
    assert _run(5000, tjdist.BLOCK)


def test_gather_with_an_empty_rank():
    assert _run(700, 1024)  # every query in block 0: rank 1 contributes nothing


def test_shard_assignment_covers_every_query_once():
    for world in (1, 2, 4, 8):
        parts = [tjdist.shard_queries(10000, i, world) for i in range(world)]
        allq = np.sort(np.concatenate(parts))
        assert (allq == np.arange(10000)).all()
        for i, p in enumerate(parts):
            assert (tjdist.shard_of(p, world) == i).all()
