"""configs[0] (GEMM 1024^3, 4096 candidates, top-64): where the small launch spends its time
(LS_TRACE phase stamps, L2 flushed before the call as in the bench), plus event timing."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_14641_b200 import workloads as W  # noqa: E402
from paper_2104_14641_b200.arch import KernelLaunch, load_arch  # noqa: E402
from paper_2104_14641_b200.engine import Task  # noqa: E402
from paper_2104_14641_b200.pack import SpaceTemplate  # noqa: E402

prog = W.program(W.matmul_json(1024))
st = SpaceTemplate(prog, W.gemm_space(1024))
task = Task(st.template.desc(load_arch("x86-avx2"), KernelLaunch.from_json(W.KERNEL_LAUNCH)), 0)
task.set_space(st.space_desc())
print("points path", task.points_path)
n = int(os.environ.get("N", "4096"))
K = int(os.environ.get("K", "64"))
d = torch.from_numpy(st.points_from_indices(W.distinct_indices(st.sizes, n, 1024)).view(np.int32)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    task.score_topk_points(d, K)
for fl in (True, False):
    ts = []
    for _ in range(20):
        if fl:
            flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        task.score_topk_points(d, K)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print("flushed" if fl else "warm", "us median", round(float(np.median(ts)), 1))
os.environ["LS_TRACE"] = "1"
flush.fill_(1)
task.score_topk_points(d, K)
torch.cuda.synchronize()
task.score_topk_points(d, K)
torch.cuda.synchronize()
