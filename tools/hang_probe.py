import sys, os
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2104_14641_b200 import workloads as W
from paper_2104_14641_b200.pack import SpaceTemplate
from paper_2104_14641_b200.arch import KernelLaunch, load_arch
from paper_2104_14641_b200 import engine as E
n = int(sys.argv[1])
st = SpaceTemplate(W.program(W.conv2d_json()), W.conv_space(4096, 1))
task = E.Task(st.template.desc(load_arch("x86-avx2"), KernelLaunch.from_json(W.KERNEL_LAUNCH)), 0)
task.set_space(st.space_desc())
pts = st.points_from_indices(W.distinct_indices(st.sizes, n, 31))
dev = torch.from_numpy(pts.view(np.int32)).cuda()
pin = torch.from_numpy(pts.view(np.int32)).pin_memory()
print("device call", flush=True)
ds, di, dn = task.score_topk_points(dev, 64, base_index=5)
torch.cuda.synchronize()
print("device ok", flush=True)
for r in range(3):
    hs, hi, hn = task.score_topk_points_host(pin, 64, base_index=5)
    print("host ok", r, hi.tolist() == di.cpu().tolist(), flush=True)
