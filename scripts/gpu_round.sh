#!/bin/bash
# Full GPU round (run under gpurun): parity suite, the driver's default bench line,
# the reference arm, then the ncu launch list + one full capture of the refinement kernels.
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo bench=$? >> gpurun_out/bench_${TAG}.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${TAG}.log 2>&1; echo ref=$? >> gpurun_out/bench_ref_${TAG}.log
[ -n "$SKIP_NCU" ] || TAG=$TAG bash scripts/profile_refine.sh
tail -3 gpurun_out/pytest_gpu.log
tail -2 gpurun_out/bench_${TAG}.log
