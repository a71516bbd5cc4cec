"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck): fused top-k in the bound merge (inline and bound_merge_kernel) and merge-tree modes,
points (device, mapped host, 3-byte) and records paths, the plain scoring kernel, the ES
generation kernels, the key merges."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_14641_b200 import engine as E  # noqa: E402
from paper_2104_14641_b200 import workloads as W  # noqa: E402
from paper_2104_14641_b200.arch import KernelLaunch, load_arch  # noqa: E402
from paper_2104_14641_b200.pack import SpaceTemplate, pack_points  # noqa: E402

st = SpaceTemplate(W.program(W.conv2d_json()), W.conv_space(512, 1))
task = E.Task(st.template.desc(load_arch("x86-avx2"), KernelLaunch.from_json(W.KERNEL_LAUNCH)), 0)
task.set_space(st.space_desc())
for n, k in [(1 << 14, 8), (1 << 14, 64), (3000, 4), (1 << 18, 64)]:  # bound K2 / tree / small / bound inline
    idx = W.distinct_indices(st.sizes, n, 5)
    pts = st.points_from_indices(idx)
    d = torch.from_numpy(pts.view(np.int32)).cuda()
    task.score_topk_points(d, k)
    task.score_points(d)
    task.score_topk_points(torch.from_numpy(pack_points(pts, 3)).cuda(), k)
    task.score_topk_points_host(torch.from_numpy(pack_points(pts, 3)).pin_memory(), k)
    if n <= 1 << 14:
        recs = st.records_from_indices(idx)
        dr = E.to_device_records(recs, 0)
        task.score_topk(dr, k)
        task.score(dr)
        task.inexact_footprints(dr)
        task.inexact_footprints(dr, notes=True)
    torch.cuda.synchronize()
run = E.EsRun(task, 0.05, 2.0, 40960, 3, 7)  # 5 sort tiles: the look-back walks
run.run()
run.result(st.dim)
run.evaluated()
run.close()
s = torch.rand(4 * 16, dtype=torch.float64, device="cuda")
i = torch.arange(4 * 16, dtype=torch.int64, device="cuda")
E.topk_merge(s, i, 4, 16, 16)
keys = torch.empty((64, 2), dtype=torch.int64, device="cuda")
E.topk_to_keys(s, i, keys)
E.topk_merge_keys(keys, 16)
torch.cuda.synchronize()
task.close()
from paper_2104_14641_b200 import code as K  # noqa: E402
from paper_2104_14641_b200.ir import parse_program  # noqa: E402
import json  # noqa: E402
prog = parse_program(json.dumps({"tensors": [{"name": "A", "dims": [8]}], "body": [
    {"loop": {"var": "i", "extent": 8, "body": [{"access": {"tensor": "A", "kind": "load", "idx": ["i"]}}]}}]}))
x86 = ("    movq $0, %r8\n.L1:\n    vmovups (%rax), %zmm0\n    vfmadd231ps %zmm0, %zmm1, %zmm2\n"
       "    vmovups %zmm2, (%rcx)\n    addq $1, %r8\n    cmpq $8, %r8\n    jne .L1\n    ret\n")
notes: list = []
K.code_features(prog, [x86, "", "    jmp nowhere\n", x86.replace("$8", "$9")], load_arch("x86-avx2"), diagnostics=notes)
K.code_features(prog, ["    mov r1, 0\nb:\n    add r1, r1, 1\n    setp.lt r1, 8\n    bra b\n",
                       "    mov r1, 1\nb:\n    mul r1, r1, 2\n    setp.lt r1, 64\n    bra b\n"],
                load_arch("nvidia-volta"), KernelLaunch.from_json(W.KERNEL_LAUNCH), diagnostics=notes)
assert any(notes), notes
torch.cuda.synchronize()
print("sanitize driver done")
