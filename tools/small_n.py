import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2104_14641_b200 import workloads as W
from paper_2104_14641_b200.engine import Task
st, desc = bench.workload("x86-avx2")
task = Task(desc, 0); task.set_space(st.space_desc())
for n in (1 << 12, 1 << 14, 1 << 16, 100_003, 1 << 18, 1 << 19, 1 << 20, 1 << 21):
    pts = st.points_from_indices(W.distinct_indices(st.sizes, n, 7))
    d = torch.from_numpy(pts.view(np.int32)).cuda()
    out = (torch.empty(64, dtype=torch.float64, device='cuda'), torch.empty(64, dtype=torch.int64, device='cuda'), torch.empty(1, dtype=torch.int64, device='cuda'))
    for _ in range(5): task.score_topk_points(d, 64, out=out)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(50): task.score_topk_points(d, 64, out=out)
    ev[1].record(); torch.cuda.synchronize()
    print("n", n, "us/call", round(ev[0].elapsed_time(ev[1]) / 50 * 1e3, 1))
