python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-baseline > gpurun_out/bench_auto.log 2>&1
tail -1 gpurun_out/bench_auto.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('auto', d['value']/1e9, d['e2e']['value']/1e9, d['roofline']['kernel_ms'])"
