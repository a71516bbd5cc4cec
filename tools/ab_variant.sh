#!/bin/bash
# A/B variant of one translation unit: tools/ab_variant.sh NAME "-DFLAG=..." [TU]
#   -> tools/ab_libs/NAME.so (TU, default k_space5.cu, recompiled with the flags and linked
#      with the other objects of the last build/)
set -e
cd "$(dirname "$0")/.."
name=$1; flags=$2; tu=${3:-k_space5.cu}
mkdir -p tools/ab_libs build/ab
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -Xcompiler -fPIC $flags \
  -c -o build/ab/$name.o paper_2104_14641_b200/csrc/$tu
objs=$(ls build/obj/*.o | grep -v "/$tu.o")
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o tools/ab_libs/$name.so build/ab/$name.o $objs
echo tools/ab_libs/$name.so
