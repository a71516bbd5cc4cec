#!/bin/bash
# A/B variant of the space path only: tools/ab_variant.sh NAME "-DFLAG=..." -> tools/ab_libs/NAME.so
# (k_space5.cu recompiled with the flags, linked with the other objects of the last build/)
set -e
cd "$(dirname "$0")/.."
name=$1; flags=$2
mkdir -p tools/ab_libs build/ab
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -Xcompiler -fPIC $flags \
  -c -o build/ab/$name.o paper_2104_14641_b200/csrc/k_space5.cu
objs=$(ls build/obj/*.o | grep -v k_space5)
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o tools/ab_libs/$name.so build/ab/$name.o $objs
echo tools/ab_libs/$name.so
