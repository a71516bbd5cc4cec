LS_HOST_TRACE=1 python - <<'PY' 2>&1 | tail -6
import sys; sys.path.insert(0, '.')
import numpy as np, torch, time, bench
from paper_2104_14641_b200 import workloads as W
from paper_2104_14641_b200.engine import Task
from paper_2104_14641_b200.pack import pack_points
st, desc = bench.workload("x86-avx2")
task = Task(desc, 0); task.set_space(st.space_desc())
pts = st.points_from_indices(W.distinct_indices(st.sizes, 1 << 20, 2104))
pin = torch.from_numpy(pack_points(pts, 3)).pin_memory()
hout = (np.empty(64, np.float64), np.empty(64, np.int64), np.zeros(1, np.int64))
for _ in range(12):
    t0 = time.perf_counter(); task.score_topk_points_host(pin, 64, out=hout); print("wall", round((time.perf_counter()-t0)*1e6, 1), file=sys.stderr)
PY
