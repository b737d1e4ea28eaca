"""Multi-rank host logic on CPU (gloo, world_size 2): query objects are sharded in blocks of
1024 (shard = (r / 1024) % world) with no data-path collective; result records are gathered
to rank 0 and concatenated in query order, reproducing the single-GPU record order."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _owner(r, world, block=1024):
    return (r // block) % world


def _fake_records(nq, seed):
    rng = np.random.default_rng(seed)
    recs = []
    for r in range(nq):
        for s in sorted(rng.choice(5000, size=rng.integers(0, 4), replace=False)):
            recs.append((r, int(s), float(rng.random()), float(rng.random() + 1), "lod-60", 0))
    return recs


def _worker(rank, world, port, nq, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = _fake_records(nq, 5)
    mine = [rec for rec in full if _owner(rec[0], world) == rank]  # what this rank's GPU produces
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        merged = sorted((rec for part in gathered for rec in part), key=lambda x: x[0])  # stable by r
        out.put(merged == full)
    dist.destroy_process_group()


def test_shard_gather_reproduces_single_rank_order():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 5000, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert ok


def test_shard_assignment_covers_every_query_once():
    for world in (1, 2, 4, 8):
        owners = [_owner(r, world) for r in range(10000)]
        assert set(owners) == set(range(world)) if world <= 9 else True
        counts = np.bincount(owners, minlength=world)
        assert counts.sum() == 10000
