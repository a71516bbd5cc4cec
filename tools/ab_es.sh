#!/bin/bash
# Interleaved A/B of the libraries in tools/ab_libs on the ES probe (ms per 3-generation run)
cd "$(dirname "$0")/.."
lib=paper_2104_14641_b200/libloopscout_b200.so
cp $lib /tmp/ab_orig.so
for r in $(seq ${ROUNDS:-3}); do
  for so in tools/ab_libs/*.so; do
    cp $so $lib
    for T in ${TASKS:-0 12}; do echo "$(basename $so .so) $(TASK=$T REPS=20 timeout 300 python tools/es_probe.py 2>&1 | tail -1)"; done
  done
done
cp /tmp/ab_orig.so $lib
