import json, sys
from collections import defaultdict, Counter
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from golden_util import GOLDEN, arch_named, launch
from paper_2104_14641_b200 import code as K
from paper_2104_14641_b200.ir import parse_program
cases = json.loads((GOLDEN / "code_analysis.json").read_text())
groups = defaultdict(list)
for i, c in enumerate(cases):
    groups[(json.dumps(c["program"], sort_keys=True), c["arch"])].append(i)
cnt = Counter(); ex = {}
for (pj, an), idx in groups.items():
    prog = parse_program(pj); arch = arch_named(an)
    res = K.code_features(prog, [cases[i]["text"] for i in idx], arch, launch())
    for i, r in zip(idx, res):
        c = cases[i]
        if "error" in c:
            ok = isinstance(r, Exception) and [type(r).__name__, str(r)] == c["error"]
            if not ok: cnt[("err", c["kind"], an)] += 1; ex.setdefault(("err", c["kind"], an), (i, c["error"], repr(r)))
            continue
        if isinstance(r, Exception):
            cnt[("raised", c["kind"], an)] += 1; ex.setdefault(("raised", c["kind"], an), (i, repr(r))); continue
        want = dict(c["features"]); got = dict(r.values)
        for k in want:
            if want[k] != got[k]:
                cnt[(k, c["kind"], an)] += 1; ex.setdefault((k, c["kind"], an), (i, got[k], want[k]))
for k, v in sorted(cnt.items()): print(k, v, ex[k])
