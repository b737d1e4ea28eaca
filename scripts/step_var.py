"""Per-step stage timings of repeated resident config-B joins (diagnoses step-time outliers)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_19982_b200 as tj  # noqa: E402
from paper_2604_19982_b200 import synth  # noqa: E402

r, s = synth.build_config("B", "/tmp/trijoin_bench/B_x1", scale=1.0)
R, S = tj.load_dataset(r), tj.load_dataset(s)
res = tj.Resident(R, S)
kw = dict(type="intersect", lods=[20, 60, 100])
if os.environ.get("SV_REFINE_CHUNK"):
    kw["refine_chunk"] = int(os.environ["SV_REFINE_CHUNK"])
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    t0 = time.perf_counter()
    o = res.run(**kw)
    wall = (time.perf_counter() - t0) * 1e3
    lv = [(l["level"], round(l["ms"], 1), round(l["kernel_ms"], 1)) for l in o["levels"]]
    print(json.dumps({"wall": round(wall, 1), "total": round(o["total_ms"], 1), "mbb": round(o["mbb_ms"], 1),
                      "voxel": round(o["voxel_ms"], 1), "levels": lv}), flush=True)
