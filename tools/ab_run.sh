#!/bin/bash
# Interleaved A/B of the libraries in tools/ab_libs (see ab_build.sh): ROUNDS x every variant.
cd "$(dirname "$0")/.."
lib=paper_2104_14641_b200/libloopscout_b200.so
cp $lib /tmp/ab_orig.so
for r in $(seq ${ROUNDS:-3}); do
  for so in tools/ab_libs/*.so; do
    cp $so $lib
    timeout 300 python bench.py --no-baseline ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "
import sys, json; d = json.loads(sys.stdin.read())
rp = d.get('records_path') or {}
print('$(basename $so .so)', round(d['value'] / 1e9, 3), round(d['e2e']['value'] / 1e9, 3) if isinstance(d.get('e2e'), dict) else None, round(d['ms_per_step'] * 1e3, 1), 'records', round(rp.get('value', 0) / 1e9, 3))"
  done
done
cp /tmp/ab_orig.so $lib
