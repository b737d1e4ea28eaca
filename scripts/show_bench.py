#!/usr/bin/env python3
"""Print ms/step and per-level counters of the last bench.py JSON line in a log."""
import json
import sys

lines = [x for x in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench.log").read().splitlines()
         if x.startswith("{")]
if not lines:
    print(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench.log").read()[-3000:])
    sys.exit(1)
d = json.loads(lines[-1])
print("ms/step", round(d["ms_per_step"], 2), "value", round(d["value"]), "frac", d.get("roofline", {}).get("frac"))
for lv in d["config"].get("levels_last_step", []):
    print({k: (round(v, 2) if isinstance(v, float) else v) for k, v in lv.items()})
