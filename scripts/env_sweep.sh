#!/bin/bash
# Bench resident joins under environment settings (tuning knobs), one line per setting:
#   SWEEP="TRIJOIN_HIER_MIN=0 TRIJOIN_HIER_MIN=1024" CONFIGS="B C" bash scripts/env_sweep.sh
mkdir -p gpurun_out
for s in ${SWEEP}; do
  for c in ${CONFIGS:-B}; do
    tag=$(echo "$s" | tr '=,' '__')
    env $(echo "$s" | tr ',' ' ') python bench.py --config $c --no-cpu-baseline --no-e2e --steps ${STEPS:-5} > gpurun_out/env_${tag}_$c.json 2> gpurun_out/env_${tag}_$c.err
    python -c "import json;d=json.load(open('gpurun_out/env_${tag}_$c.json'));print('$s', '$c', round(d['ms_per_step'],2), [(l['level'], round(l['kernel_ms'],2), round(l.get('screen_ms',0),2), l['tested']) for l in d['config']['levels_last_step']])" || tail -3 gpurun_out/env_${tag}_$c.err
  done
done
