python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
for mb in 4 3; do
  sed -i "s/return mode == 5 ? [34] : mode ? 3/return mode == 5 ? $mb : mode ? 3/" paper_2104_14641_b200/csrc/engine.cu
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$mb.log 2>&1
  timeout 300 python bench.py --no-baseline > gpurun_out/bench_mb$mb.log 2>&1
  tail -1 gpurun_out/bench_mb$mb.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('mb$mb', d['value']/1e9, d['e2e']['value']/1e9, d['roofline']['kernel_ms'])"
  python tools/trace_topk.py 2>&1 | grep LS_TRACE | tail -1 | cut -c1-150
done
