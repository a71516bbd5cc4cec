"""Where the end-to-end (host-buffer) call spends its time: device vs mapped-host points, traced."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2104_14641_b200 import engine as E  # noqa: E402
from paper_2104_14641_b200 import workloads as W  # noqa: E402
from paper_2104_14641_b200.engine import Task  # noqa: E402
from paper_2104_14641_b200.pack import pack_points  # noqa: E402

st, desc = bench.workload("x86-avx2")
task = Task(desc, 0)
task.set_space(st.space_desc())
pts = st.points_from_indices(W.distinct_indices(st.sizes, 1 << 20, 2104))
dev = torch.from_numpy(pts.view(np.int32)).cuda()
pin = torch.from_numpy(pack_points(pts, 3)).pin_memory()
pin4 = torch.from_numpy(pts.view(np.int32)).pin_memory()
hout = (np.empty(64, np.float64), np.empty(64, np.int64), np.zeros(1, np.int64))
calls = (("device", lambda: task.score_topk_points(dev, 64)),
         ("host 3B", lambda: task.score_topk_points_host(pin, 64, out=hout)),
         ("host 4B", lambda: task.score_topk_points_host(pin4, 64, out=hout)))
for _ in range(5):
    for _, fn in calls:
        fn()
torch.cuda.synchronize()
for name, fn in calls:
    ts = []
    for _ in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(name, "wall us median", round(1e6 * float(np.median(ts)), 1))
L = E.lib()
s_, i_, nv_ = hout
args = (task._h, pin.data_ptr(), 3, pin.shape[0], 0, 64, s_.ctypes.data, i_.ctypes.data, nv_.ctypes.data, None)
ts = []
for _ in range(20):
    t0 = time.perf_counter()
    L.ls_score_topk_points_host(*args)
    ts.append(time.perf_counter() - t0)
print("raw C-ABI host call (3B) wall us median", round(1e6 * float(np.median(ts)), 1))
# GPU-side span of the raw host call (events around it on the legacy stream) vs its wall time
ts, gs = [], []
for _ in range(30):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(torch.cuda.default_stream())
    t0 = time.perf_counter()
    L.ls_score_topk_points_host(*args)
    t1 = time.perf_counter()
    b.record(torch.cuda.default_stream())
    torch.cuda.synchronize()
    ts.append(t1 - t0)
    gs.append(a.elapsed_time(b) * 1e-3)
print("raw call wall us", round(1e6 * float(np.median(ts)), 1), "| GPU span event->event us", round(1e6 * float(np.median(gs)), 1))
os.environ["LS_TRACE"] = "1"
task.score_topk_points(dev, 64)
task.score_topk_points_host(pin, 64, out=hout)
torch.cuda.synchronize()
