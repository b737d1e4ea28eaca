#!/bin/bash
# ncu launch list of one resident join + one full capture of a chosen kernel launch.
mkdir -p gpurun_out
TAG=${TAG:-p}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --profile > gpurun_out/launches_${TAG}.log 2>&1
if [ -n "$NCU_K" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${NCU_K}" --launch-skip ${NCU_SKIP:-0} -c ${NCU_COUNT:-1} \
    -o gpurun_out/prof_${TAG} python bench.py --profile > gpurun_out/prof_${TAG}.log 2>&1
fi
tail -2 gpurun_out/launches_${TAG}.log | cut -c 1-400
