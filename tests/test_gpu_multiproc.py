"""Multi-GPU paths on one B200 (the only GPU the build has): several query shards in one
process (TRIJOIN_DEVICES=0,0,0: one host thread + context per shard, each uploading only its
own queries), combined with out-of-core R chunks, and one process per shard (as under
torchrun: TRIJOIN_PROCESS_SHARD=i/2, two processes on GPU 0 joined by a gloo group) with the
records gathered to rank 0 by paper_2604_19982_b200.dist. Everything must reproduce the
reference's records and stage counters exactly."""
import json
import os
import socket
import subprocess
import sys

import pytest

import tjtest
from tjtest import golden

pytestmark = pytest.mark.gpu

JOINS = [j for j in tjtest.golden_joins() if j["r"] in ("nuclei60", "mini18_s21", "spheres80a")]


def _paths(j):
    return golden(j["r"] + ".idx"), (golden(j["s"] + ".idx") if j["s"] else "")


def _stages(out):
    return [{k: v for k, v in st.items() if k != "wall_ms"} for st in out["stats"]["stages"]]


@pytest.mark.parametrize("env", [{"TRIJOIN_DEVICES": "0,0,0", "TRIJOIN_SHARD_BLOCK": "5"},
                                 {"TRIJOIN_DEVICES": "0,0", "TRIJOIN_SHARD_BLOCK": "3", "TRIJOIN_R_CHUNK_OBJECTS": "4"}],
                         ids=["3threads", "2threads_chunked"])
@pytest.mark.parametrize("j", JOINS, ids=tjtest.join_id)
def test_threaded_shards_match_reference(monkeypatch, env, j):
    import paper_2604_19982_b200 as tj
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    r, s = _paths(j)
    out = tj.join(r, s, **j["kwargs"])
    assert out["records"] == j["records"]
    assert _stages(out) == j["stages"]
    assert out["stats"]["b200"]["devices"] == len(env["TRIJOIN_DEVICES"].split(","))


def test_threaded_shards_upload_only_their_queries(monkeypatch):
    """Each shard thread uploads only its own queries: R crosses PCIe once in total while S is
    replicated to every context (before: every GPU received all of R)."""
    from paper_2604_19982_b200 import _core
    R = _core.load_dataset(golden("nuclei60.idx"))
    S = _core.load_dataset(golden("vessels8.idx"))
    kw = dict(type="within", tau=0.5, lods=[20, 60, 100])

    def h2d(a, b):
        return json.loads(_core.join_datasets(a, b, **kw)[1])["b200"]["h2d_bytes"]
    r_bytes, s_bytes = h2d(R, R), h2d(S, S)  # self-joins ship one dataset once
    monkeypatch.setenv("TRIJOIN_DEVICES", "0,0,0,0")
    monkeypatch.setenv("TRIJOIN_SHARD_BLOCK", "4")
    four = h2d(R, S)
    assert four <= 1.05 * r_bytes + 4 * s_bytes + 4096
    assert four < 4 * r_bytes


WORKER = r"""
import json, os, sys
import numpy as np
import torch.distributed as dist
sys.path.insert(0, os.environ["TJ_ROOT"])
from paper_2604_19982_b200 import _core, dist as tjdist
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
os.environ["TRIJOIN_PROCESS_SHARD"] = f"{rank}/{world}"
dist.init_process_group("gloo", rank=rank, world_size=world)
kw = json.loads(os.environ["TJ_KW"])
R = _core.load_dataset(os.environ["TJ_R"])
S = _core.load_dataset(os.environ["TJ_S"]) if os.environ["TJ_S"] else R
try:
    recs, stats = _core.join_datasets(R, S, records="array", **kw)
    merged = tjdist.gather_records(recs)
    st = tjdist.gather_stats(stats)
    if rank == 0:
        out = {"records": [[x[0], x[1], float(x[2]).hex(), float(x[3]).hex(), x[4], x[5]]
                           for x in tjdist.records_to_tuples(merged)],
               "stages": [{k: v for k, v in s.items() if k != "wall_ms"} for s in st["stages"]],
               "mine": int(len(recs))}
        with open(os.environ["TJ_OUT"], "w") as f:
            json.dump(out, f)
finally:
    dist.destroy_process_group()
"""


@pytest.mark.parametrize("j", [j for j in JOINS if j["r"] in ("nuclei60", "mini18_s21")], ids=tjtest.join_id)
def test_two_process_shards_gather_to_reference(tmp_path, j):
    """Two processes, one query shard each (TRIJOIN_PROCESS_SHARD), records gathered to rank 0
    with the product's gather: identical records, order and summed stage counters."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r, sp = _paths(j)
    kw = dict(j["kwargs"])
    outp = str(tmp_path / "out.json")
    procs = []
    for rank in range(2):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   TJ_ROOT=tjtest.ROOT, TJ_R=r, TJ_S=sp, TJ_KW=json.dumps(kw), TJ_OUT=outp,
                   TRIJOIN_SHARD_BLOCK="4", TRIJOIN_DEVICES="0")
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER], env=env))
    for p in procs:
        assert p.wait(timeout=300) == 0
    got = json.load(open(outp))
    want = [[x[0], x[1], float(x[2]).hex(), float(x[3]).hex(), x[4], x[5]] for x in j["records"]]
    assert got["records"] == want
    assert got["stages"] == j["stages"]
