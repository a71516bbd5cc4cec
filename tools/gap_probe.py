import sys, os
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2104_14641_b200 import workloads as W
from paper_2104_14641_b200.engine import Task
st, desc = bench.workload("x86-avx2")
task = Task(desc, 0); task.set_space(st.space_desc())
n = 1 << 20
pts = st.points_from_indices(W.distinct_indices(st.sizes, n, 2104))
d = torch.from_numpy(pts.view(np.int32)).cuda()
out = (torch.empty(64, dtype=torch.float64, device='cuda'), torch.empty(64, dtype=torch.int64, device='cuda'), torch.empty(1, dtype=torch.int64, device='cuda'))
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
for _ in range(5): task.score_topk_points(d, 64, out=out)
torch.cuda.synchronize()
for mode in ("flush", "noflush", "back2back"):
    ts = []
    for rep in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if mode == "flush": flush.zero_()
        a.record()
        task.score_topk_points(d, 64, out=out)
        b.record()
        if mode != "back2back": torch.cuda.synchronize()
        ts.append((a, b))
    torch.cuda.synchronize()
    print(mode, [round(a.elapsed_time(b) * 1e3, 1) for a, b in ts])
# an empty kernel's event-to-event time for scale
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
x = torch.empty(1, device='cuda')
a.record(); x.add_(1); b.record(); torch.cuda.synchronize(); print("tiny torch kernel", round(a.elapsed_time(b)*1e3, 1))
