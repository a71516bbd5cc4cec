# iteration: build, GPU parity, bench (auto path), one ncu --set full of the fused kernel
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
tail -3 gpurun_out/bench.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:score_topk_kernel -s 3 -c 1 -o gpurun_out/topk_full python bench.py --steps 2 --warmup 1 --no-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
