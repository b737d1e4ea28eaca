"""Timeline of repeated e2e config-B joins (join_datasets: host datasets in, records out)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_19982_b200 as tj  # noqa: E402
from paper_2604_19982_b200 import _core, synth  # noqa: E402

r, s = synth.build_config("B", "/tmp/trijoin_bench/B_x1", scale=1.0)
R, S = tj.load_dataset(r), tj.load_dataset(s)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    t0 = time.perf_counter()
    recs, js = _core.join_datasets(R, S, type="intersect", lods=[20, 60, 100])
    wall = (time.perf_counter() - t0) * 1e3
    st = json.loads(js)
    tl = sorted(st["b200"]["timeline"].items(), key=lambda x: x[1] if "arena" not in x[0] else -1)
    print(round(wall, 1), [(k, round(v, 1)) for k, v in tl if "arena" not in k], flush=True)
    b = st["b200"]
    print("   b200", {k: (round(v, 2) if isinstance(v, float) else v) for k, v in b.items() if k.endswith("_ms")}, flush=True)
    lv = st["b200"].get("levels", [])
    print("   levels", [(l.get("level"), round(l.get("ms", 0), 1), round(l.get("wait_ms", 0), 1)) for l in lv], flush=True)
