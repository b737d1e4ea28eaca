#!/bin/bash
# ncu --set full captures of every hot kernel of one resident config-B join (one launch each)
# plus the launch list; summaries are made in the build container (scripts/ncu_table.py).
mkdir -p gpurun_out
TAG=${TAG:-n}
run() { # name regex skip count
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" --launch-skip $3 -c $4 \
    -o gpurun_out/ncu_${TAG}_$1 python bench.py --profile > gpurun_out/ncu_${TAG}_$1.log 2>&1
}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --profile > gpurun_out/launches_${TAG}.log 2>&1
run filters "k_mbb_count|k_mbb_fill|k_vf_bounds|k_vf_scatter|k_prep|k_seg_prep|k_aggregate" 0 9
# one refinement launch per level and pass (launch size >= 16Mi voxel pairs): k_screen / k_seed
# launch i = LOD level i; k_eval: seed and screen evaluations alternate (LOD-60 screen = 3)
run screen60 "k_screen" 1 1
run screen100 "k_screen" 2 1
run seed60 "k_seed" 1 1
run eval60 "k_eval" 3 1
ls gpurun_out | grep ncu_${TAG}
