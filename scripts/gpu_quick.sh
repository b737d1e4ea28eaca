#!/bin/bash
# Quick GPU check (run under gpurun): parity suite + a config-B bench without the CPU/e2e legs.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/bench.log
tail -3 gpurun_out/pytest_gpu.log
