python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
python - <<'PY'
import sys; sys.path.insert(0, '.')
import bench
from paper_2104_14641_b200.engine import Task
st, desc = bench.workload("x86-avx2"); t = Task(desc, 0); t.set_space(st.space_desc()); print("conv points path", t.points_path)
PY
timeout 300 python bench.py --no-baseline > gpurun_out/bench_auto.log 2>&1
tail -1 gpurun_out/bench_auto.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('auto', d['value']/1e9, d['e2e']['value']/1e9, d['roofline']['kernel_ms'])"
timeout 600 python bench.py --workload bert --steps 10 > gpurun_out/bench_bert.log 2>&1; tail -1 gpurun_out/bench_bert.log | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 python tools/trace_topk.py > gpurun_out/ncu_k2.log 2>&1
grep -E "gpu__time" gpurun_out/ncu_k2.log | tail -4
