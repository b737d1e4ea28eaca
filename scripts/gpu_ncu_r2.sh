#!/bin/bash
# ncu evidence of one resident config-B join (bench.py --profile): the launch list,
# --set full captures of the filter / compaction kernels (HBM roofline rows) and of the
# LOD-100 refinement launches (k_screen with source lines, k_seed, k_eval).
mkdir -p gpurun_out
TAG=${TAG:-r2}
ARGS=${ARGS:-}
run() { # name regex skip count
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" --launch-skip $3 -c $4 \
    -o gpurun_out/ncu_${TAG}_$1 python bench.py --profile $ARGS > gpurun_out/ncu_${TAG}_$1.log 2>&1
}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --profile $ARGS > gpurun_out/launches_${TAG}.log 2>&1
run filters "k_mbb_count|k_mbb_fill|k_vf_bounds|k_vf_scatter|k_gather_sorted" 0 5
run compact "k_tile_select|k_tile_sums|k_tile_scan" 0 3
run screen100 "k_screen" 2 1
run seed100 "k_seed" 5 1   # decision mode: 2 seed launches per level (primary, rest)
run eval100 "k_eval" 7 1   # 3 per level: primary seeds, other seeds, screen
ls gpurun_out | grep ncu_${TAG}
