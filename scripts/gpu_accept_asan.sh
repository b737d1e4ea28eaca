#!/bin/bash
# The reference acceptance harness against an AddressSanitizer build of the drop-in
# (variants/asan: host code instrumented; diagnostics for a crash at exit).
mkdir -p gpurun_out
export ASAN_OPTIONS=protect_shadow_gap=0:detect_leaks=0:halt_on_error=1:replace_intrin=0:verify_asan_link_order=0
timeout 2400 variants/asan/acceptance_asan > gpurun_out/acceptance_asan.log 2> gpurun_out/acceptance_asan.err
echo "asan acceptance rc=$?"; tail -2 gpurun_out/acceptance_asan.log; head -60 gpurun_out/acceptance_asan.err
