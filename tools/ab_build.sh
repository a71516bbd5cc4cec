#!/bin/bash
# A/B builds: tools/ab_build.sh NAME [git-rev] -> tools/ab_libs/NAME.so (working tree when no rev).
# tools/ab_run.sh then benches every variant interleaved on one box (same clocks, same host).
set -e
cd "$(dirname "$0")/.."
name=$1; rev=$2
src=paper_2104_14641_b200/csrc
if [ -n "$rev" ]; then
  d=$(mktemp -d); mkdir -p $d/pkg/csrc; ln -s "$PWD/include" $d/include  # engine.cu includes ../../include
  for f in engine.cu es.cuh blocksched.cpp; do git show "$rev:$src/$f" > "$d/pkg/csrc/$f"; done
  src=$d/pkg/csrc
fi
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -Xcompiler -fPIC -shared \
  -Iinclude -o tools/ab_libs/$name.so $src/engine.cu $src/blocksched.cpp
echo tools/ab_libs/$name.so
