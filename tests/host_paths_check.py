"""Run by tests/test_engine_gpu.py (LS_HOST_PATH is read once per process): host-buffer points
calls == device calls over several (n, k, point width), pinned and pageable."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_14641_b200 import workloads as W  # noqa: E402
from paper_2104_14641_b200.arch import KernelLaunch, load_arch  # noqa: E402
from paper_2104_14641_b200.engine import Task  # noqa: E402
from paper_2104_14641_b200.pack import SpaceTemplate, pack_points  # noqa: E402

st = SpaceTemplate(W.program(W.conv2d_json()), W.conv_space(4096, 1))
task = Task(st.template.desc(load_arch("x86-avx2"), KernelLaunch.from_json(W.KERNEL_LAUNCH)), 0)
task.set_space(st.space_desc())
pts_all = st.points_from_indices(W.distinct_indices(st.sizes, (1 << 20) + 777, 61))
bad = []
for n, k in [((1 << 20) + 777, 64), (1 << 16, 16), (100_003, 64), (300_001, 200), (5000, 8)]:
    pts = pts_all[:n]
    d = torch.from_numpy(pts.view(np.int32)).cuda()
    ds, di, dn = task.score_topk_points(d, k, base_index=3)
    torch.cuda.synchronize()
    want_i, want_s, want_n = di.cpu().tolist(), ds.cpu().numpy(), int(dn.item())
    for host in (pack_points(pts, 3), pts.view(np.uint32).copy()):
        for pinned in (True, False):
            h = torch.from_numpy(host).pin_memory() if pinned else host
            for rep in range(2):
                hs, hi, hn = task.score_topk_points_host(h, k, base_index=3)
                if not (hi.tolist() == want_i and np.array_equal(hs, want_s) and hn == want_n):
                    bad.append((n, k, host.shape, pinned, rep))
task.close()
print("BAD" if bad else "OK", bad)
sys.exit(1 if bad else 0)
