#!/bin/bash
# Bench config B with each library build under variants/<name>/ (kernel tuning experiments).
mkdir -p gpurun_out
cp paper_2604_19982_b200/libtrijoin_b200.so /tmp/lib_base.so
for v in $(ls variants); do
  cp variants/$v/libtrijoin_b200.so paper_2604_19982_b200/libtrijoin_b200.so
  for c in ${CONFIGS:-B}; do
    python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 ${ARGS} > gpurun_out/var_${v}_$c.json 2> gpurun_out/var_${v}_$c.err
    python -c "import json;d=json.load(open('gpurun_out/var_${v}_$c.json'));print('$v', '$c', round(d['ms_per_step'],2), [(l['level'], round(l['kernel_ms'],2)) for l in d['config']['levels_last_step']])"
  done
done
cp /tmp/lib_base.so paper_2604_19982_b200/libtrijoin_b200.so
