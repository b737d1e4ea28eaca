"""Host-side logic that runs without a GPU: the C-ABI library loads and exports its header,
index I/O round-trips the reference's bytes, spec validation errors, benchmark placement."""
import ctypes
import json
import os
import shutil

import numpy as np
import pytest

import tjtest
from tjtest import golden


def test_capi_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(tjtest.LIB)
    names = tjtest.capi_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_capi_without_gpu_fails_loudly_not_silently():
    lib = tjtest.load_capi()
    ctx = ctypes.c_void_p()
    rc = lib.tj_ctx_create(0, ctypes.byref(ctx))
    if rc == 0:  # a GPU is present: nothing to check here
        lib.tj_ctx_destroy(ctx)
        pytest.skip("GPU present")
    assert rc in (1, 3)
    assert lib.tj_global_last_error()


def test_host_dataset_view_matches_index(tmp_path):
    lib = tjtest.load_capi()
    h = ctypes.c_void_p()
    assert lib.tj_host_dataset_load(golden("mini12_s31.idx").encode(), ctypes.byref(h)) == 0
    v = lib.tj_host_dataset_view(h).contents
    assert v.n_objects == 12 and v.n_levels == 5
    assert [v.levels[i] for i in range(5)] == [20, 40, 60, 80, 100]
    nv = v.voxel_offsets[12]
    # every level's CSR covers all facets of every object exactly once (voxel partition)
    fo = v.facet_offsets[4]
    assert fo[nv] > 0
    assert lib.tj_host_dataset_bytes(h) > 0
    lib.tj_host_dataset_free(h)
    assert lib.tj_host_dataset_load(str(tmp_path / "missing.idx").encode(), ctypes.byref(h)) != 0


def test_index_roundtrip_is_byte_identical(tmp_path):
    """load_index + save_index (this library's own 3DPJ1 code) reproduce the reference's bytes."""
    from paper_2604_19982_b200 import _core
    src = golden("mini9_s13_vr15.idx")
    ds = _core.load_dataset(src)
    out = tmp_path / "copy.idx"
    _core.save_dataset(ds, str(out))
    a = open(src, "rb").read()
    b = open(out, "rb").read()
    assert a == b


@pytest.mark.parametrize("cut", [3, 100, -9])
def test_index_corruption_raises(tmp_path, cut):
    from paper_2604_19982_b200 import _core
    data = open(golden("mini12_s31.idx"), "rb").read()
    bad = tmp_path / "bad.idx"
    bad.write_bytes(data[:cut] if cut > 0 else data + b"\0" * 9)
    with pytest.raises(Exception) as e:
        _core.load_dataset(str(bad))
    assert "index" in str(e.value).lower()


def test_bad_magic(tmp_path):
    from paper_2604_19982_b200 import _core
    bad = tmp_path / "bad.idx"
    bad.write_bytes(b"XXXXX" + b"\0" * 64)
    with pytest.raises(Exception, match="bad magic"):
        _core.load_dataset(str(bad))


@pytest.mark.parametrize("kw", [dict(tau=-1.0), dict(type="knn", k=0), dict(type="nearest"),
                                dict(type="intersect", tau=0.5), dict(filter_chunk=0), dict(refine_chunk=0),
                                dict(lods=[20, 40]), dict(lods=[40, 20, 100]), dict(lods=[0, 100])])
def test_invalid_spec_raises_value_error(kw):
    """proj/python/tests/test_smoke.py:70-76 and validate() (proj/src/engine.cpp:38-56); raised
    before any device work, so this runs on CPU."""
    import paper_2604_19982_b200 as tj
    with pytest.raises(ValueError):
        tj.join(golden("mini12_s31.idx"), **kw)


def test_scatter_targets_match_reference_generator(ref_module, tmp_path):
    """synth.scatter_targets reproduces generate(scatter_within=...)'s per-object placement
    (proj/src/dataset.cpp:183-190): object centres equal the SplitMix64 targets."""
    from paper_2604_19982_b200 import synth
    box = (0.0, 0.0, 0.0, 41.6, 41.6, 41.6)
    gen = ref_module.generate(str(tmp_path / "g"), shape="sphere", facets=300, scale=0.35, count=50, seed=21,
                              scatter_within=box)
    targets = synth.scatter_targets(21, 50, box)
    centres = []
    for f in gen["files"]:
        v, _ = ref_module.parse_off(open(tmp_path / "g" / f).read())
        v = np.asarray(v)
        centres.append((v.min(0) + v.max(0)) / 2)
    np.testing.assert_allclose(np.asarray(centres), targets, atol=1e-12)


def test_replicated_objects_are_translated_templates(tmp_path):
    from paper_2604_19982_b200 import _core, synth
    r, s = synth.build_config("B", str(tmp_path), scale=0.0005)
    ds = _core.load_dataset(r)
    assert ds.n_objects == 50 and ds.lod_schedule == [20, 60, 100]
    tmpl = _core.load_dataset(os.path.join(synth.BENCHDATA, "sphere300_s035.idx"))
    assert ds.facet_count(2) == sum(1 for _ in range(50)) * (tmpl.facet_count(2) // tmpl.n_objects)
