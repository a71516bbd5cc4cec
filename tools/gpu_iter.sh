# iteration: build, GPU parity, A/B bench, one ncu --set full of the fused kernel
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --path 1 --no-baseline > gpurun_out/bench_p1.log 2>&1; echo b1=$?
timeout 300 python bench.py --path 2 --no-baseline > gpurun_out/bench_p2.log 2>&1; echo b2=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:score_topk_kernel -s 3 -c 1 -o gpurun_out/topk_full python bench.py --steps 2 --warmup 1 --no-baseline --path 2 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
grep -h '"value"' gpurun_out/bench_p*.log | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['config']['arch'], d['value']/1e9, d['e2e']['value']/1e9, d['roofline']['kernel_ms'])"
