# every bench line (BASELINE configs[0..4] + the reference arm) into gpurun_out/bench_<w>.json
for w in conv gemm bert resnet50-es sweep; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w rc=$?"
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
