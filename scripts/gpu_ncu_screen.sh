#!/bin/bash
# ncu --set full capture (source-correlated) of one k_screen launch of a resident config-B join
# (default: the LOD-100 launch, the third); TAG names the report.
mkdir -p gpurun_out
TAG=${TAG:-screen}
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${KERNEL:-k_screen}" --launch-skip ${SKIP:-2} -c 1 \
    -o gpurun_out/ncu_${TAG} python bench.py --profile ${ARGS} > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_${TAG}.log
