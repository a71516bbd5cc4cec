# Round-2 evidence: GPU tests, every bench line, the launch list, one ncu --set full of the fused
# kernel (+ source page), compute-sanitizer logs.  Outputs in gpurun_out/ (copied to profiles/).
set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02b.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r02b.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02b.txt 2>&1
bash tools/gpu_bench_all.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02b.csv python bench.py --steps 4 --warmup 3 --no-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:score_topk_kernel<.int.3, .int.4, .int.5, .int.1>" -s 2 -c 1 -o gpurun_out/pts_full_r02b \
  python bench.py --steps 2 --warmup 1 --no-baseline > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/pts_full_r02b.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/pts_src_r02b.csv 2>/dev/null
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_driver.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer_$tool.txt
done
tail -n 2 gpurun_out/pytest_gpu_r02b.txt
