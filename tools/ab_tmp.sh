for cs in 1 0; do
  sed -i "s/^#define TOPK_CAP_SMALL [01]/#define TOPK_CAP_SMALL $cs/" paper_2104_14641_b200/csrc/engine.cu
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$cs.log 2>&1
  timeout 300 python bench.py --no-baseline > gpurun_out/bench_cs$cs.log 2>&1
  tail -1 gpurun_out/bench_cs$cs.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cap_small=$cs', d['value']/1e9, d['e2e']['value']/1e9, d['roofline']['kernel_ms'])"
  python tools/trace_topk.py 2>&1 | grep "LS_TRACE n" | tail -2 | cut -c1-120
done
