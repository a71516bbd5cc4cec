"""Per-task timing + phase trace of the BERT bench tasks (configs[3])."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_14641_b200 import workloads as W  # noqa: E402
from paper_2104_14641_b200.arch import KernelLaunch, load_arch  # noqa: E402
from paper_2104_14641_b200.engine import Task  # noqa: E402
from paper_2104_14641_b200.pack import SpaceTemplate  # noqa: E402

for j, (name, spec, space) in enumerate(W.bert_tasks()):
    st = SpaceTemplate(W.program(spec), space)
    task = Task(st.template.desc(load_arch("x86-avx2"), KernelLaunch.from_json(W.KERNEL_LAUNCH)), 0)
    task.set_space(st.space_desc())
    n = min(838860, int(st.size))
    pts = st.points_from_indices(W.distinct_indices(st.sizes, n, 40 + j))
    d = torch.from_numpy(pts.view(np.int32)).cuda()
    for _ in range(3):
        task.score_topk_points(d, 64)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        task.score_topk_points(d, 64)
    torch.cuda.synchronize()
    print(name, "sizes", list(st.sizes), "path", task.points_path, "us/call", round((time.perf_counter() - t0) / 10 * 1e6, 1),
          flush=True)
    os.environ["LS_TRACE"] = "1"
    task.score_topk_points(d, 64)
    torch.cuda.synchronize()
    os.environ.pop("LS_TRACE")
    task.close()
