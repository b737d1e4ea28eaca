#!/bin/bash
# Builds variants/<name>/libtrijoin_b200.so: refine.cu recompiled with extra flags, linked with
# the other objects of the current build (run `make -C paper_2604_19982_b200/csrc` first).
# usage: scripts/build_variant.sh <name> [-DFOO=1 ...]; bench them with scripts/variants.sh
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2604_19982_b200/csrc"
mkdir -p ../../variants/$name build/var
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC \
    -Xcompiler -ffp-contract=off -I../../include -Xptxas -warn-spills "$@" -c refine.cu -o build/var/refine_$name.o 2>&1 \
    | grep -o "k_screenILb[01].*spill.*\|error.*" || true
objs=$(ls build/*.o | grep -v '/refine.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../../variants/$name/libtrijoin_b200.so \
    $objs build/var/refine_$name.o -lpthread
echo "built variants/$name"
