"""Run by tests/test_engine_gpu.py::test_topk_merge_modes_forced in a child process (LS_MERGE is
read once per process): every (n, k) through the fused top-k under the forced merge mode must equal
a stable sort of the same candidates' scores."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_14641_b200 import workloads as W  # noqa: E402
from paper_2104_14641_b200.arch import KernelLaunch, load_arch  # noqa: E402
from paper_2104_14641_b200.engine import Task  # noqa: E402
from paper_2104_14641_b200.pack import SpaceTemplate  # noqa: E402

st = SpaceTemplate(W.program(W.conv2d_json()), W.conv_space(4096, 1))
task = Task(st.template.desc(load_arch("x86-avx2"), KernelLaunch.from_json(W.KERNEL_LAUNCH)), 0)
task.set_space(st.space_desc())
pts_all = st.points_from_indices(W.distinct_indices(st.sizes, 1 << 20, 41))
bad = []
for n, k in [(1 << 20, 64), (100_003, 64), (1 << 18, 16), (1 << 16, 64), (1 << 19, 111), (5000, 8), (1 << 20, 1)]:
    d = torch.from_numpy(pts_all[:n].view(np.int32)).cuda()
    s, _, _ = task.score_points(d, features=False)
    for rep in range(2):
        ts, ti, nv = task.score_topk_points(d, k, base_index=7)
        torch.cuda.synchronize()
        sc = s.cpu().numpy()
        want = np.lexsort((np.arange(n), sc))[:k]
        ok = (ti.cpu().numpy() - 7).tolist() == want.tolist() and np.array_equal(ts.cpu().numpy(), sc[want]) \
            and int(nv.item()) == int(np.isfinite(sc).sum())
        if not ok:
            bad.append((n, k, rep))
task.close()
print("BAD" if bad else "OK", bad)
sys.exit(1 if bad else 0)
