#!/bin/bash
# ncu evidence for the refinement kernels (run under gpurun; outputs to gpurun_out/).
#   1. launch list of one full resident join (every kernel with its device time; cold, serialised)
#   2. one `--set full` capture of the screen and exact-evaluation kernels with source correlation
SCALE=${SCALE:-1}
TAG=${TAG:-r1}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --profile --scale ${SCALE} > gpurun_out/launches_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${KERNELS:-k_screen|k_eval}" \
    --launch-skip ${NCU_SKIP:-0} -c ${NCU_COUNT:-4} \
    -o gpurun_out/prof_${TAG} python bench.py --profile --scale ${SCALE} > gpurun_out/prof_${TAG}.log 2>&1
