# parity suite on the working-tree library, then interleaved A/B of tools/ab_libs/*.so, then a trace per variant
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
ROUNDS=${ROUNDS:-3} bash tools/ab_run.sh
lib=paper_2104_14641_b200/libloopscout_b200.so
cp $lib /tmp/ab_orig2.so
for so in tools/ab_libs/*.so; do
  cp $so $lib
  echo "== trace $(basename $so .so)"
  LS_TRACE=1 timeout 300 python tools/trace_topk.py 2>&1 | grep LS_TRACE | sed -n '2,3p;5,6p'
done
cp /tmp/ab_orig2.so $lib
for so in tools/ab_libs/*.so; do cp $so $lib; echo "== small n $(basename $so .so)"; timeout 300 python tools/small_n.py; done
cp /tmp/ab_orig2.so $lib
