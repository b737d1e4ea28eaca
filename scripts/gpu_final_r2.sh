#!/bin/bash
# Round-2 bench lines of every BASELINE configuration with the current build (profiles/), the
# reference arm for B, and the reference acceptance harness against the drop-in.
mkdir -p gpurun_out
export TRIJOIN_BACKTRACE=1
run() { # tag args...
  local tag=$1; shift
  timeout 1500 python bench.py "$@" > gpurun_out/final_$tag.json 2> gpurun_out/final_$tag.err
  echo "$tag rc=$? $(python scripts/show_bench.py gpurun_out/final_$tag.json 2>/dev/null | head -3)"
}
run B
run B_ref --impl reference
run A --config A --cpu-stride 1
run C --config C --cpu-stride 400 --steps 3
run D --config D --steps 3 --cpu-stride 1000
run E --config E --steps 3 --cpu-stride 100
timeout 1500 tests/cpp/acceptance_dropin > gpurun_out/final_acceptance.log 2>&1; echo "acceptance rc=$? $(tail -1 gpurun_out/final_acceptance.log)"
free -g | head -2
