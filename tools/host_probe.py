"""Host-side cost of one ls_score_topk_points call (Python wrapper vs raw C-ABI), and the
device step with and without the host launch latency inside the timed region."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2104_14641_b200 import workloads as W  # noqa: E402
from paper_2104_14641_b200.engine import Task, lib  # noqa: E402

st, desc = bench.workload("x86-avx2")
task = Task(desc, 0)
task.set_space(st.space_desc())
n, k = 1 << 20, 64
pts = st.points_from_indices(W.distinct_indices(st.sizes, n, 2104))
d = torch.from_numpy(pts.view(np.int32)).cuda()
out = (torch.empty(k, dtype=torch.float64, device="cuda"), torch.empty(k, dtype=torch.int64, device="cuda"),
       torch.empty(1, dtype=torch.int64, device="cuda"))
for _ in range(10):
    task.score_topk_points(d, k)
torch.cuda.synchronize()
L = lib()
sp = torch.cuda.current_stream().cuda_stream
args = (task._h, d.data_ptr(), 4, n, 0, k, out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(), sp)
for name, fn in (("python wrapper", lambda: task.score_topk_points(d, k)),
                 ("python wrapper, out=", lambda: task.score_topk_points(d, k, out=out)),
                 ("raw ctypes", lambda: L.ls_score_topk_points(*args))):
    hs = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(100):
            fn()
        hs.append((time.perf_counter() - t0) / 100)
        torch.cuda.synchronize()
    # one call after an idle GPU: host call time alone (returns before the GPU finishes)
    one = []
    for _ in range(50):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        one.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    # events: synchronous step (record, call, record) vs back-to-back steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
    for a, b in ev:
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    sync_ms = np.median([a.elapsed_time(b) for a, b in ev])
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{name:22s} host us/call (queued) {1e6 * min(hs):6.1f}  first call after idle {1e6 * np.median(one):6.1f}  "
          f"event step us {1e3 * sync_ms:6.1f}  back-to-back us/step {1e3 * a.elapsed_time(b) / 50:6.1f}")
