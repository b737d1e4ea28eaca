#!/bin/bash
# GPU suite, then e2e config-B joins with R's last level shipped whole vs in pieces.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not acceptance" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for p in 0 1; do
  echo "TRIJOIN_PIECED=$p"
  TRIJOIN_PIECED=$p TRIJOIN_DEBUG_TIMELINE=1 timeout 600 python scripts/e2e_timeline.py 5 2>&1 | grep -v "^   levels" | tail -6
done
