"""Per-kernel breakdown of one ES task (run under ncu --metrics gpu__time_duration.sum)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_14641_b200 import workloads as W
from paper_2104_14641_b200.arch import KernelLaunch, load_arch
from paper_2104_14641_b200.engine import EsRun, Task
from paper_2104_14641_b200.pack import SpaceTemplate

gens = int(os.environ.get("GENS", "3"))
pop = int(os.environ.get("POP", str(1 << 20)))
which = int(os.environ.get("TASK", "0"))
name, spec, space = W.resnet50_tasks()[which]
st = SpaceTemplate(W.program(spec), space)
task = Task(st.template.desc(load_arch(os.environ.get("ARCH", "x86-avx2")), KernelLaunch.from_json(W.KERNEL_LAUNCH)), 0)
task.set_space(st.space_desc())
run = EsRun(task, 0.05, 2.0, pop, gens, 2104)
run.run()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(int(os.environ.get("REPS", "5"))):
    run.run()
torch.cuda.synchronize()
print(name, task.points_path, "ms/run", (time.perf_counter() - t) * 1e3 / int(os.environ.get("REPS", "5")))
