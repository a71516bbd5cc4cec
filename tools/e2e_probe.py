"""Where the end-to-end (host-buffer) call spends its time: device vs mapped-host points, traced."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2104_14641_b200 import workloads as W  # noqa: E402
from paper_2104_14641_b200.engine import Task  # noqa: E402

st, desc = bench.workload("x86-avx2")
task = Task(desc, 0)
task.set_space(st.space_desc())
pts = st.points_from_indices(W.distinct_indices(st.sizes, 1 << 20, 2104))
dev = torch.from_numpy(pts.view(np.int32)).cuda()
pin = torch.from_numpy(pts.view(np.int32)).pin_memory()
for _ in range(5):
    task.score_topk_points(dev, 64)
    task.score_topk_points_host(pin, 64)
torch.cuda.synchronize()
for name, fn in (("device", lambda: task.score_topk_points(dev, 64)), ("host", lambda: task.score_topk_points_host(pin, 64))):
    ts = []
    for _ in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(name, "wall us median", 1e6 * float(np.median(ts)))
os.environ["LS_TRACE"] = "1"
task.score_topk_points(dev, 64)
task.score_topk_points_host(pin, 64)
torch.cuda.synchronize()
