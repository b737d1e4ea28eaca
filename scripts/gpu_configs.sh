#!/bin/bash
# Bench lines for the other BASELINE configurations (profiles only; the driver's line is B).
mkdir -p gpurun_out
TAG=${TAG:-c}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest=$? >> gpurun_out/pytest_${TAG}.log
timeout 900 python bench.py --config C --steps 3 --cpu-stride 400 > gpurun_out/bench_C_${TAG}.log 2>&1; echo rc=$? >> gpurun_out/bench_C_${TAG}.log
timeout 900 python bench.py --config E --scale 0.02 --steps 3 --cpu-stride 20 > gpurun_out/bench_E_${TAG}.log 2>&1; echo rc=$? >> gpurun_out/bench_E_${TAG}.log
timeout 900 python bench.py --config A --steps 3 --cpu-stride 1 > gpurun_out/bench_A_${TAG}.log 2>&1; echo rc=$? >> gpurun_out/bench_A_${TAG}.log
df -h /tmp | tail -1 > gpurun_out/disk_${TAG}.log; free -g >> gpurun_out/disk_${TAG}.log; nproc >> gpurun_out/disk_${TAG}.log
