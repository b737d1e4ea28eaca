#!/bin/bash
# Iteration check (run under gpurun): GPU parity suite (without the 4-minute reference acceptance
# harness) and resident-join benches of the configs in $CONFIGS (default B C).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not acceptance" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-B C}; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --steps ${STEPS:-5} ${ARGS} > gpurun_out/it_$c.json 2> gpurun_out/it_$c.err
  python -c "import json;d=json.load(open('gpurun_out/it_$c.json'));print('$c', round(d['ms_per_step'],2), [(l['level'], round(l['kernel_ms'],2), l['tested'], l['screened'], l['evaluated']) for l in d['config']['levels_last_step']])" || tail -5 gpurun_out/it_$c.err
done
