"""Compact-resident datasets (TJ_DATASET_COMPACT): every level stays in HBM in
the shipped compact mesh form and a join expands, per level, only the voxels its active voxel
pairs touch, in chunks of a working-set budget. This is what lets inputs whose expanded form
exceeds HBM (SURVEY configs D and E) run on one B200. Results must be identical to the
reference's: every golden join, the adversarial culling cases, --exact, k-NN, forced tiny
working sets (many chunks per level), and combined with query shards and R chunks."""
import json

import pytest

import tjtest
from tjtest import golden

pytestmark = pytest.mark.gpu

JOINS = tjtest.golden_joins()
ADVERSARIAL = tjtest.adversarial_joins()


def _paths(j):
    return golden(j["r"] + ".idx"), (golden(j["s"] + ".idx") if j["s"] else "")


def _check(out, j):
    assert out["records"] == j["records"]
    assert [{k: v for k, v in st.items() if k != "wall_ms"} for st in out["stats"]["stages"]] == j["stages"]
    assert out["stats"]["b200"]["residency"] == "compact"


@pytest.mark.parametrize("j", JOINS, ids=tjtest.join_id)
def test_compact_matches_reference(monkeypatch, j):
    import paper_2604_19982_b200 as tj
    monkeypatch.setenv("TRIJOIN_COMPACT", "1")
    r, s = _paths(j)
    _check(tj.join(r, s, **j["kwargs"]), j)


@pytest.mark.parametrize("j", [j for j in JOINS if j["r"] in ("nuclei60", "mini18_s21", "spheres80a")],
                         ids=tjtest.join_id)
def test_compact_tiny_working_set(monkeypatch, j):
    """A 50 kB working set splits the levels' active voxel pairs into many expansions (down to
    single voxel pairs)."""
    import paper_2604_19982_b200 as tj
    monkeypatch.setenv("TRIJOIN_COMPACT", "1")
    monkeypatch.setenv("TRIJOIN_WORKSET_MB", "0.05")
    r, s = _paths(j)
    out = tj.join(r, s, **j["kwargs"])
    _check(out, j)
    if j["r"] == "nuclei60":  # several expansions per level (3 levels)
        assert out["stats"]["b200"]["mat_chunks"] > 3


@pytest.mark.parametrize("j", ADVERSARIAL, ids=tjtest.join_id)
def test_compact_adversarial(monkeypatch, j):
    import paper_2604_19982_b200 as tj
    monkeypatch.setenv("TRIJOIN_COMPACT", "1")
    monkeypatch.setenv("TRIJOIN_WORKSET_MB", "2")
    r, s = _paths(j)
    _check(tj.join(r, s, **j["kwargs"]), j)


@pytest.mark.parametrize("j", [j for j in JOINS if j["r"] in ("nuclei60", "mini18_s21")], ids=tjtest.join_id)
def test_compact_with_shards_and_r_chunks(monkeypatch, j):
    import paper_2604_19982_b200 as tj
    for k, v in {"TRIJOIN_COMPACT": "1", "TRIJOIN_DEVICES": "0,0", "TRIJOIN_SHARD_BLOCK": "3",
                 "TRIJOIN_R_CHUNK_OBJECTS": "5", "TRIJOIN_WORKSET_MB": "4"}.items():
        monkeypatch.setenv(k, v)
    r, s = _paths(j)
    _check(tj.join(r, s, **j["kwargs"]), j)


def test_compact_chosen_by_budget(monkeypatch):
    """With a device budget below the expanded footprint the engine switches to compact
    residency by itself (no override) and stays exact."""
    import paper_2604_19982_b200 as tj
    j = next(j for j in JOINS if j["r"] == "nuclei60" and j["kwargs"]["type"] == "within")
    monkeypatch.setenv("TRIJOIN_DEVICE_BUDGET_MB", "70")
    r, s = _paths(j)
    _check(tj.join(r, s, **j["kwargs"]), j)


def test_resident_compact_equals_expanded():
    """The bench's device-resident handle in compact mode: same candidates and counters."""
    from paper_2604_19982_b200 import _core
    R = _core.load_dataset(golden("nuclei60.idx"))
    S = _core.load_dataset(golden("vessels8.idx"))
    kw = dict(type="within", tau=0.5, lods=[20, 60, 100], arrays=True)
    a = _core.Resident(R, S).run(**kw)
    b = _core.Resident(R, S, compact=True).run(**kw)
    for key in ("n_cands", "confirmed", "voxel_pairs_in", "vp_generated", "vp_pruned"):
        assert a[key] == b[key]
    for key in ("pair_r", "pair_s", "status", "decided_at"):
        assert (a[key] == b[key]).all()
    assert (tjtest.bits(a["lb"]) == tjtest.bits(b["lb"])).all()
    assert (tjtest.bits(a["ub"]) == tjtest.bits(b["ub"])).all()


@pytest.mark.parametrize("cfg,scale", [("B", 0.01), ("E", 0.0004)])
def test_compact_benchmark_scale_matches_reference(ref_module, monkeypatch, tmp_path, cfg, scale):
    import paper_2604_19982_b200 as tj
    from paper_2604_19982_b200 import synth
    monkeypatch.setenv("TRIJOIN_COMPACT", "1")
    r, s = synth.build_config(cfg, str(tmp_path), scale=scale)
    kw = dict(synth.CONFIGS[cfg][2], lods=synth.LODS)
    a = ref_module.join(r, s, **kw)
    b = tj.join(r, s, **kw)
    assert [tuple(map(repr, x)) for x in a["records"]] == [tuple(map(repr, x)) for x in b["records"]]
    strip = lambda st: [{k: v for k, v in x.items() if k != "wall_ms"} for x in st["stages"]]
    assert strip(a["stats"]) == strip(b["stats"])
