#!/bin/bash
# The reference acceptance harness (proj/tests/acceptance.cpp) against the drop-in, with native
# backtraces and ThreadPool integrity checks (diagnostics).
mkdir -p gpurun_out
TRIJOIN_POOL_CHECK=1 TRIJOIN_BACKTRACE=1 timeout 1500 stdbuf -o0 tests/cpp/acceptance_dropin > gpurun_out/acceptance.log 2> gpurun_out/acceptance.err
echo "acceptance rc=$?"; tail -2 gpurun_out/acceptance.log; grep -v "^  " gpurun_out/acceptance.err | head -40
