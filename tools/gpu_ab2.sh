# interleaved A/B of tools/ab_libs/*.so (bench value) + a 2^20 / 2^22 trace per variant
ROUNDS=${ROUNDS:-3} bash tools/ab_run.sh
lib=paper_2104_14641_b200/libloopscout_b200.so
cp $lib /tmp/ab_orig3.so
for so in tools/ab_libs/*.so; do
  cp $so $lib
  echo "== trace $(basename $so .so)"
  LS_TRACE=1 timeout 300 python tools/trace_topk.py 2>&1 | grep LS_TRACE | sed -n '3p;6p' | cut -c1-120
done
cp /tmp/ab_orig3.so $lib
