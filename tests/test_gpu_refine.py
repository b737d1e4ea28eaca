"""tj_refine_batch (backs refine_kernel, proj/src/refine.cpp:63-84) through the C-ABI, bitwise
against the reference kernel's per-voxel-pair bounds at every level (the logic of
proj/tests/test_refine.cpp:92-146, dumped by the reference in tests/golden/staged_*.bin)."""
import ctypes

import numpy as np
import pytest

import tjtest
from tjtest import bits, golden

pytestmark = pytest.mark.gpu


def _view(capi, path):
    h = ctypes.c_void_p()
    assert capi.lib.tj_host_dataset_load(path.encode(), ctypes.byref(h)) == 0
    return h, capi.lib.tj_host_dataset_view(h).contents


def _gather(vr_view, vs_view, cands, active, level):
    """Build (tris, hd, ph, descriptors) for `active` at `level` from the packed CSR views."""
    li_r = [vr_view.levels[i] for i in range(vr_view.n_levels)].index(level)
    li_s = [vs_view.levels[i] for i in range(vs_view.n_levels)].index(level)
    tris, hd, ph, ro, so, rl, sl = [], [], [], [], [], [], []
    n = 0

    def seg(view, li, obj, v):
        nonlocal n
        g = view.voxel_offsets[obj] + v
        b, e = view.facet_offsets[li][g], view.facet_offsets[li][g + 1]
        rec = np.ctypeslib.as_array(view.facets[li], (max(e, 1) * 12,))[b * 12:e * 12].reshape(-1, 12)
        tris.append(rec[:, :9])
        hd.append(rec[:, 9])
        ph.append(rec[:, 10])
        off = n
        n += e - b
        return off, e - b

    for op, vr, vs in active:
        r, s = int(cands["r"][op]), int(cands["s"][op])
        a, la = seg(vr_view, li_r, r, vr)
        b, lb = seg(vs_view, li_s, s, vs)
        ro.append(a), rl.append(la), so.append(b), sl.append(lb)
    cat = (lambda xs: np.concatenate(xs)) if tris else (lambda xs: np.zeros(0))
    return (np.concatenate(tris).reshape(-1, 9), cat(hd), cat(ph), np.array(ro, np.uint64), np.array(so, np.uint64),
            np.array(rl, np.uint32), np.array(sl, np.uint32))


@pytest.mark.parametrize("flags", [0, 1], ids=["cull", "nocull"])
@pytest.mark.parametrize("dump", ["staged_mini10_s61.bin", "staged_nuclei60_vs_vessels8.bin"])
def test_refine_batch_bitexact_every_level(capi, dump, flags):
    cands, active, levels = tjtest.load_staged(golden(dump))
    r_name, s_name = ("mini10_s61", "mini10_s61") if "mini10" in dump else ("nuclei60", "vessels8")
    hr, vr = _view(capi, golden(r_name + ".idx"))
    hs, vs = _view(capi, golden(s_name + ".idx"))
    try:
        for level, fp, ref_lb, ref_ub in levels:
            tris, hd, ph, ro, so, rl, sl = _gather(vr, vs, cands, active, level)
            assert int((rl.astype(np.uint64) * sl).sum()) == fp  # reference facet-pair count
            lb, ub = capi.refine_batch(tris, hd, ph, ro, so, rl, sl, flags=flags)
            assert (bits(lb) == bits(ref_lb)).all(), f"level {level}"
            assert (bits(ub) == bits(ref_ub)).all(), f"level {level}"
            assert (lb >= 0).all()
            if level == 100:  # hd = ph = 0 at level 100: lb == ub == exact voxel-pair distance
                assert (bits(lb) == bits(ub)).all()
    finally:
        capi.lib.tj_host_dataset_free(hr)
        capi.lib.tj_host_dataset_free(hs)


def test_refine_batch_empty_segments(capi):
    """Empty segments give (+inf, +inf) (proj/src/refine.cpp:66-67)."""
    tris = np.random.default_rng(1).uniform(-1, 1, (4, 9))
    z = np.zeros(4)
    lb, ub = capi.refine_batch(tris, z, z, [0, 0, 2], [2, 2, 2], [0, 2, 2], [2, 0, 2])
    assert np.isinf(lb[0]) and np.isinf(ub[0]) and np.isinf(lb[1]) and np.isinf(ub[1])
    assert np.isfinite(lb[2])
