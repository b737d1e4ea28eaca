"""Full join parity on the GPU: records and stage statistics equal the reference's on the
same inputs (tests/golden/joins.json, produced by the reference), through the Python drop-in
(-> C++ run_join -> C-ABI tj_join) and directly through the C-ABI; plus invariances,
sharding and error behaviour (proj/tests/test_engine.cpp, proj/python/tests/test_smoke.py)."""
import os

import numpy as np
import pytest

import tjtest
from tjtest import golden

pytestmark = pytest.mark.gpu

JOINS = tjtest.golden_joins()


def _paths(j):
    return golden(j["r"] + ".idx"), (golden(j["s"] + ".idx") if j["s"] else "")


@pytest.mark.parametrize("j", JOINS, ids=tjtest.join_id)
def test_join_matches_reference_records_and_stats(j):
    import paper_2604_19982_b200 as tj
    r, s = _paths(j)
    out = tj.join(r, s, **j["kwargs"])
    assert out["records"] == j["records"]
    stages = [{k: v for k, v in st.items() if k != "wall_ms"} for st in out["stats"]["stages"]]
    assert stages == j["stages"]
    assert out["stats"]["query"] == j["query"] and out["stats"]["results"] == j["results"]


@pytest.mark.parametrize("j", JOINS[::3], ids=tjtest.join_id)
def test_join_through_capi(capi, j):
    r, s = _paths(j)
    kw = dict(j["kwargs"])
    R = capi.load(r)
    S = capi.load(s) if s else R
    try:
        c = capi.join(R, S, **kw)
        assert tjtest.records_from_candidates(c, kw["type"] == "knn") == j["records"]
    finally:
        capi.free(R)
        if s:
            capi.free(S)


@pytest.mark.parametrize("refine_chunk", [1, 100, 500000])
def test_chunk_and_cull_invariance(capi, refine_chunk):
    """Results are independent of the refine launch size and of culling (test_refine.cpp:183-218)."""
    R = capi.load(golden("mini10_s61.idx"))
    try:
        base = capi.join(R, R, type="within", tau=1.3, flags=1)
        for flags in (0, 1):
            c = capi.join(R, R, type="within", tau=1.3, flags=flags, refine_chunk=refine_chunk)
            for key in ("pair_r", "pair_s", "status", "decided_at"):
                assert (c[key] == base[key]).all()
            assert (tjtest.bits(c["lb"]) == tjtest.bits(base["lb"])).all()
            assert (tjtest.bits(c["ub"]) == tjtest.bits(base["ub"])).all()
    finally:
        capi.free(R)


OUT_OF_CORE = [j for j in JOINS if j["r"] in ("nuclei60", "mini18_s21", "mini10_s77", "spheres80a")]


@pytest.mark.parametrize("env", [{"TRIJOIN_R_CHUNK_OBJECTS": "7"},
                                 {"TRIJOIN_DEVICE_BUDGET_MB": "70", "TRIJOIN_COMPACT": "0"},
                                 {"TRIJOIN_DEVICE_BUDGET_MB": "66"}],
                         ids=["chunk7", "budget70MB_expanded", "budget66MB_auto"])
@pytest.mark.parametrize("j", OUT_OF_CORE, ids=tjtest.join_id)
def test_out_of_core_r_chunks(monkeypatch, env, j):
    """R joined in consecutive object chunks against a resident S (device-memory budget,
    SURVEY §8d config D): records and every stage counter equal the reference's."""
    import paper_2604_19982_b200 as tj
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    r, s = _paths(j)
    out = tj.join(r, s, **j["kwargs"])
    assert out["records"] == j["records"]
    stages = [{k: v for k, v in st.items() if k != "wall_ms"} for st in out["stats"]["stages"]]
    assert stages == j["stages"]
    b = out["stats"]["b200"]
    if j["r"] == "nuclei60":  # chunked, unless compact residency made it fit
        assert b["r_chunks"] > 1 or (b["residency"] == "compact" and "TRIJOIN_COMPACT" not in env)


@pytest.mark.parametrize("order", ["1", "0"], ids=["ordered", "unordered"])
@pytest.mark.parametrize("pieced", ["1", "2", "0"], ids=["pieced", "pieced_all", "whole"])
@pytest.mark.parametrize("j", [j for j in JOINS if j["s"]], ids=tjtest.join_id)
def test_pieced_last_level(monkeypatch, j, pieced, order):
    """R's last join level shipped in object-range pieces (the default; TRIJOIN_PIECED=2: every
    join level after the first, each piece refined with R's running level aggregates; 0: whole;
    tj_dataset_set_pieced / tj_dataset_finish_level_part), the join refining each piece's queries
    as it lands, with and without the cross-dataset copy order (TRIJOIN_COPY_ORDER,
    tj_dataset_copy_after): records and every stage counter equal the reference's."""
    import paper_2604_19982_b200 as tj
    monkeypatch.setenv("TRIJOIN_PIECED", pieced)
    monkeypatch.setenv("TRIJOIN_COPY_ORDER", order)
    r, s = _paths(j)
    out = tj.join(r, s, **j["kwargs"])
    assert out["records"] == j["records"]
    stages = [{k: v for k, v in st.items() if k != "wall_ms"} for st in out["stats"]["stages"]]
    assert stages == j["stages"]


@pytest.mark.parametrize("j", [j for j in JOINS if j["r"] in ("nuclei60", "spheres80a")], ids=tjtest.join_id)
def test_process_shards_partition_the_queries(monkeypatch, j):
    """One process per GPU (bench.py under torchrun): TRIJOIN_PROCESS_SHARD=i/n joins the
    query blocks of shard i only; the shards' records partition the full result."""
    import paper_2604_19982_b200 as tj
    r, s = _paths(j)
    monkeypatch.setenv("TRIJOIN_SHARD_BLOCK", "7")
    got = []
    for i in range(3):
        monkeypatch.setenv("TRIJOIN_PROCESS_SHARD", f"{i}/3")
        got += tj.join(r, s, **j["kwargs"])["records"]
    monkeypatch.delenv("TRIJOIN_PROCESS_SHARD")
    assert sorted(got) == sorted(j["records"])


@pytest.mark.parametrize("idx", ["mini10_s61.idx", "mini18_s21.idx", "spheres80a.idx"])
def test_intersect_decision_mode(capi, idx):
    """Intersection joins refine in decision mode unless TJ_FLAG_EXACT_INTERVALS (4): statuses
    and stages are identical to the exhaustive run; confirmed intervals are bit-identical (the
    only intervals an intersection's records carry); with the flag every interval is."""
    R = capi.load(golden(idx))
    try:
        lods = (20, 60, 100)
        base = capi.join(R, R, type="intersect", lods=lods, flags=1 | 4)
        dec = capi.join(R, R, type="intersect", lods=lods)
        exact = capi.join(R, R, type="intersect", lods=lods, flags=4)
        assert dec["decision_mode"] == 1 and exact["decision_mode"] == 0
        for c in (dec, exact):
            for key in ("pair_r", "pair_s", "status", "decided_at"):
                assert (c[key] == base[key]).all()
        conf = base["status"] == 1
        for key in ("lb", "ub"):
            assert (tjtest.bits(dec[key][conf]) == tjtest.bits(base[key][conf])).all()
            assert (tjtest.bits(exact[key]) == tjtest.bits(base[key])).all()
    finally:
        capi.free(R)


@pytest.mark.parametrize("idx", ["mini10_s61.idx", "mini18_s21.idx", "spheres80a.idx"])
def test_decision_mode_tripwire_sample(capi, monkeypatch, idx):
    """Decision mode keeps exact intervals on a sample of ops ($TRIJOIN_TRIPWIRE_SAMPLE, every
    N-th op; default 1024), so the reference's bound-crossing tripwire (src/filter.cpp:22-32)
    is evaluated on them. With N = 1 every op's interval equals the exact-interval run."""
    R = capi.load(golden(idx))
    try:
        lods = (20, 60, 100)
        exact = capi.join(R, R, type="intersect", lods=lods, flags=4)
        monkeypatch.setenv("TRIJOIN_TRIPWIRE_SAMPLE", "1")
        dec = capi.join(R, R, type="intersect", lods=lods)
        assert dec["decision_mode"] == 1
        for key in ("pair_r", "pair_s", "status", "decided_at"):
            assert (dec[key] == exact[key]).all()
        assert (tjtest.bits(dec["lb"]) == tjtest.bits(exact["lb"])).all()
        assert (tjtest.bits(dec["ub"]) == tjtest.bits(exact["ub"])).all()
        monkeypatch.setenv("TRIJOIN_TRIPWIRE_SAMPLE", "4")  # every 4th op exact, the rest decision
        part = capi.join(R, R, type="intersect", lods=lods)
        every4 = (np.arange(len(part["lb"])) % 4) == 0
        assert (tjtest.bits(part["lb"][every4]) == tjtest.bits(exact["lb"][every4])).all()
        for key in ("pair_r", "pair_s", "status", "decided_at"):
            assert (part[key] == exact[key]).all()
    finally:
        capi.free(R)


@pytest.mark.parametrize("kw", [dict(type="within", tau=0.9), dict(type="knn", k=3)])
def test_shards_merge_to_single_run(capi, kw):
    """R-sharded runs (query blocks across GPUs, no data-path collective) merge to
    exactly the single-device candidate set."""
    R = capi.load(golden("mini18_s21.idx"))
    try:
        full = capi.join(R, R, **kw)
        parts = [capi.join(R, R, shard=(i, 3), **kw) for i in range(3)]
        # block size 1024 > |R| puts every query on shard 0; exercise it anyway
        merged = {k: np.concatenate([p[k] for p in parts]) for k in ("pair_r", "pair_s", "status", "lb")}
        order = np.lexsort((merged["pair_s"], merged["pair_r"]))
        for k in ("pair_r", "pair_s", "status"):
            assert (merged[k][order] == full[k]).all()
        assert (tjtest.bits(merged["lb"][order]) == tjtest.bits(full["lb"])).all()
    finally:
        capi.free(R)


def test_self_join_keeps_identity_pairs():
    """proj/python/tests/test_smoke.py:33-46; proj/README.md:99-101."""
    import paper_2604_19982_b200 as tj
    out = tj.join(golden("mini12_s31.idx"), tau=1.0)
    pairs = {(r, s) for r, s, *_ in out["records"]}
    assert all((i, i) in pairs for i in range(12))
    for r, s, lb, ub, stage, rank in out["records"]:
        assert lb <= ub <= 1.0 + 1e-9 and rank == 0
    for st in out["stats"]["stages"]:
        assert st["pairs_in"] - st["confirmed"] - st["removed"] == st["pairs_out"]


def test_intersect_equals_within_zero():
    import paper_2604_19982_b200 as tj
    a = tj.join(golden("mini12_s31.idx"), type="intersect")
    b = tj.join(golden("mini12_s31.idx"), type="within", tau=0.0)
    assert a["records"] == b["records"] and a["stats"]["query"] == "intersect"


def test_knn_ranks():
    import paper_2604_19982_b200 as tj
    out = tj.join(golden("mini14_s53.idx"), type="knn", k=2)
    by_r = {}
    for r, s, lb, ub, stage, rank in out["records"]:
        by_r.setdefault(r, []).append(rank)
    assert len(by_r) == 14 and all(sorted(v) == [1, 2] for v in by_r.values())


def test_missing_lod_is_engine_error():
    """A join level absent from a dataset's schedule is an EngineError (src/refine.cpp:16-21)."""
    import paper_2604_19982_b200 as tj
    with pytest.raises(RuntimeError, match="not in the dataset's lod schedule"):
        tj.join(golden("nuclei60.idx"), golden("vessels8.idx"), tau=0.5, lods=[20, 40, 100])


def test_empty_inputs(capi, tmp_path):
    """A join whose MBB stage finds nothing (tau = 0, far apart objects) and an empty R."""
    import paper_2604_19982_b200 as tj
    from paper_2604_19982_b200 import _core
    out = tj.join(golden("nuclei60.idx"), golden("spheres80a.idx"), tau=0.0, lods=[20, 60, 100])
    assert out["stats"]["results"] == len(out["records"])
    empty = tmp_path / "empty.idx"
    _core.replicate_index(_core.load_dataset(golden("nuclei60.idx")), str(empty), [], [])
    out = tj.join(str(empty), golden("vessels8.idx"), tau=1.0, lods=[20, 60, 100])
    assert out["records"] == [] and out["stats"]["stages"][0]["pairs_in"] == 0


@pytest.mark.parametrize("cfg,scale", [("B", 0.002), ("C", 0.0005), ("A", 0.02), ("D", 0.0001), ("E", 0.001)])
def test_benchmark_configs_match_reference(ref_module, tmp_path, cfg, scale):
    """Scaled benchmark configurations (same density) against the live reference build."""
    import paper_2604_19982_b200 as tj
    from paper_2604_19982_b200 import synth
    r, s = synth.build_config(cfg, str(tmp_path), scale=scale)
    kw = dict(synth.CONFIGS[cfg][2], lods=synth.LODS)
    a = ref_module.join(r, s, **kw)
    b = tj.join(r, s, **kw)
    assert a["records"] == b["records"]
    strip = lambda st: [{k: v for k, v in x.items() if k != "wall_ms"} for x in st["stages"]]
    assert strip(a["stats"]) == strip(b["stats"])


ADVERSARIAL = tjtest.adversarial_joins()


@pytest.mark.parametrize("j", ADVERSARIAL, ids=tjtest.join_id)
def test_adversarial_culling_matches_reference(j):
    """Near-parallel faces / edges at gaps 1e-12 .. 1e-2 and sliver facets (sin ~ 5e-3 .. 1.7e-2)
    at coordinates around +-100 (tests/golden/make_adversarial.py): the exact-preserving culling
    margins (refine_kernel.cuh) must leave records and every stage counter equal to the
    reference's."""
    import paper_2604_19982_b200 as tj
    r, s = _paths(j)
    out = tj.join(r, s, **j["kwargs"])
    assert out["records"] == j["records"]
    stages = [{k: v for k, v in st.items() if k != "wall_ms"} for st in out["stats"]["stages"]]
    assert stages == j["stages"]


@pytest.mark.parametrize("j", [j for j in ADVERSARIAL if j["kwargs"]["type"] in ("intersect", "within")
                               and not j["kwargs"].get("exact")], ids=tjtest.join_id)
def test_adversarial_intervals_bitwise_vs_no_cull(capi, j):
    """Every candidate interval (not only the records) equals the exhaustive evaluation's
    (culling off), with exact intervals on: the culling skipped nothing that mattered."""
    r, s = _paths(j)
    R = capi.load(r)
    S = capi.load(s) if s else R
    try:
        kw = dict(j["kwargs"])
        lods = tuple(kw.pop("lods"))
        base = capi.join(R, S, lods=lods, flags=1 | 4, **kw)
        c = capi.join(R, S, lods=lods, flags=4, **kw)
        for key in ("pair_r", "pair_s", "status", "decided_at"):
            assert (c[key] == base[key]).all()
        assert (tjtest.bits(c["lb"]) == tjtest.bits(base["lb"])).all()
        assert (tjtest.bits(c["ub"]) == tjtest.bits(base["ub"])).all()
    finally:
        capi.free(R)
        if s:
            capi.free(S)


@pytest.mark.parametrize("kw", [dict(type="within", tau=0.5), dict(type="knn", k=3), dict(type="intersect"),
                                dict(type="within", tau=0.5, exact=True)])
def test_exact_queue_overflow_rerun(capi, monkeypatch, kw):
    """A level whose exact-evaluation queue overflows is re-run with a larger queue
    (refine_loop.cu): forced here with a 16-slot queue; results are bit-identical."""
    R = capi.load(golden("nuclei60.idx"))
    S = capi.load(golden("vessels8.idx"))
    try:
        lods = (20, 60, 100)
        base = capi.join(R, S, lods=lods, **kw)
        assert base["queue_reruns"] == 0
        monkeypatch.setenv("TRIJOIN_TEST_QUEUE_CAP", "16")
        c = capi.join(R, S, lods=lods, **kw)
        assert c["queue_reruns"] > 0
        for key in ("pair_r", "pair_s", "status", "decided_at"):
            assert (c[key] == base[key]).all()
        assert (tjtest.bits(c["lb"]) == tjtest.bits(base["lb"])).all()
        assert (tjtest.bits(c["ub"]) == tjtest.bits(base["ub"])).all()
    finally:
        capi.free(R)
        capi.free(S)


@pytest.mark.parametrize("cfg,scale", [("B", 0.02), ("D", 0.001), ("C", 0.005)])
def test_benchmark_scale_matches_reference(ref_module, tmp_path, cfg, scale):
    """Larger slices of the benchmark configurations (B: 2k x 2k nuclei, ~7k candidate pairs;
    D: 1k x 1k at tau 0.2; C: 1k nuclei x 50 vessels k-NN) against the live reference build:
    every record bit for bit (repr of the doubles) and every stage counter."""
    import paper_2604_19982_b200 as tj
    from paper_2604_19982_b200 import synth
    r, s = synth.build_config(cfg, str(tmp_path), scale=scale)
    kw = dict(synth.CONFIGS[cfg][2], lods=synth.LODS)
    a = ref_module.join(r, s, **kw)
    b = tj.join(r, s, **kw)
    assert len(a["records"]) > 100
    assert [tuple(map(repr, x)) for x in a["records"]] == [tuple(map(repr, x)) for x in b["records"]]
    strip = lambda st: [{k: v for k, v in x.items() if k != "wall_ms"} for x in st["stages"]]
    assert strip(a["stats"]) == strip(b["stats"])
