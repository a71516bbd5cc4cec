"""Phase timestamps of the fused kernel (LS_TRACE=1) on the bench workload, printed by the library."""
import os
import sys
from pathlib import Path

os.environ["LS_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2104_14641_b200 import workloads as W  # noqa: E402
from paper_2104_14641_b200.engine import Task  # noqa: E402

st, desc = bench.workload("x86-avx2")
task = Task(desc, 0)
task.set_space(st.space_desc())
for n in [int(x) for x in os.environ.get("TRACE_N", str((1 << 20)) + "," + str(1 << 22)).split(",")]:
    pts = st.points_from_indices(W.distinct_indices(st.sizes, n, 2104))
    d = torch.from_numpy(pts.view(np.int32)).cuda()
    for _ in range(3):
        task.score_topk_points(d, 64)
    torch.cuda.synchronize()
