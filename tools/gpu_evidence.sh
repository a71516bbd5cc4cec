# round evidence: GPU tests, smoke, headline bench (+ reference arm), extra workloads,
# launch list of the headline command, one ncu --set full of the fused points kernel
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 300 python bench.py --arch nvidia-volta --no-baseline > gpurun_out/bench_volta.log 2>&1; echo volta=$?
timeout 600 python bench.py --workload bert --steps 10 > gpurun_out/bench_bert.log 2>&1; echo bert=$?
timeout 900 python bench.py --workload resnet50-es --steps 3 --warmup 3 > gpurun_out/bench_res.log 2>&1; echo res=$?
timeout 900 python bench.py --workload sweep --steps 8 > gpurun_out/bench_sweep.log 2>&1; echo sweep=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:score_topk_kernel<.int.3, .int.4, .int.5, .int.1>" -s 2 -c 1 -o gpurun_out/pts_full_r01 \
  python bench.py --steps 2 --warmup 1 --no-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
ncu -i gpurun_out/pts_full_r01.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/pts_src_r01.csv 2>/dev/null
for f in bench bench_ref bench_volta bench_bert bench_res bench_sweep; do tail -n 1 gpurun_out/$f.log | cut -c1-300; done
LS_TRACE=1 timeout 100 python -m pytest tests/test_engine_gpu.py -q -s -k workspace_reuse 2>&1 | grep -o "LS_TRACE n=[0-9]* grid=[0-9]*\|survivors [0-9]*" | paste - - > gpurun_out/reuse_survivors.txt
timeout 120 python tools/host_probe.py > gpurun_out/host_probe.txt 2>&1
