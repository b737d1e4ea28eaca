#!/bin/bash
# Parity suite + bench without the CPU leg (e2e included); optional ncu of one kernel.
mkdir -p gpurun_out
TAG=${TAG:-x}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu_${TAG}.log
timeout 900 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_${TAG}.log 2>&1; echo bench=$? >> gpurun_out/bench_${TAG}.log
if [ -n "$NCU_K" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${NCU_K}" --launch-skip ${NCU_SKIP:-0} -c ${NCU_COUNT:-1} \
    -o gpurun_out/prof_${TAG} python bench.py --profile > gpurun_out/prof_${TAG}.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu_${TAG}.log
tail -2 gpurun_out/bench_${TAG}.log | cut -c 1-3000
