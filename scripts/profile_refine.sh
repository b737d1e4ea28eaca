#!/bin/bash
# ncu evidence for the refinement kernel (run under gpurun; outputs to gpurun_out/).
#   1. launch list of one full join (every kernel with its device time; cold, serialised)
#   2. one `--set full` capture of refine_join_kernel with source correlation
set -e
SCALE=${SCALE:-0.02}
TAG=${TAG:-r1}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --profile --scale ${SCALE} > gpurun_out/launches_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:refine_join_kernel -c ${NCU_COUNT:-2} \
    -o gpurun_out/prof_${TAG} python bench.py --profile --scale ${SCALE} > gpurun_out/prof_${TAG}.log 2>&1
