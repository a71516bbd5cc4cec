# build, GPU parity, A/B bench of the points paths (auto = space-specialised), launch list
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-baseline > gpurun_out/bench_auto.log 2>&1; echo b0=$?
timeout 300 python bench.py --path 2 --no-baseline > gpurun_out/bench_p2.log 2>&1; echo b2=$?
timeout 300 python bench.py --no-baseline --arch nvidia-volta > gpurun_out/bench_v.log 2>&1; echo bv=$?
grep -h '"value"' gpurun_out/bench_auto.log gpurun_out/bench_p2.log gpurun_out/bench_v.log | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['config']['arch'], d['path'], 'value', d['value']/1e9, 'e2e', d['e2e']['value']/1e9, 'kms', d['roofline']['kernel_ms'], 'rec', d['records_path']['value']/1e9)"
