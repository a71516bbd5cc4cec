# quick iteration: GPU parity suite, headline bench, phase trace (library prebuilt in-tree)
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('value', d['value']/1e9, 'e2e', d['e2e']['value']/1e9, 'ms', d['ms_per_step'], 'sync_ms', d.get('sync_step_ms'), 'kern_ms', d['roofline']['kernel_ms'], 'rec', d['records_path']['value']/1e9)"
LS_TRACE_BLOCKS=1 timeout 300 python tools/trace_topk.py > gpurun_out/trace.log 2>&1; echo trace=$?
grep -v blocks gpurun_out/trace.log | head -8
