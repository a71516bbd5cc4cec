"""Aggregate an ncu source page (cuda,sass CSV) by enclosing CUDA function: thread instructions per candidate.

    python tools/ncu_funcs.py src.csv n_candidates
The source text is taken from the report itself, so it matches the profiled build.
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
ncand = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr]
ti = h.index("Thread Instructions Executed")
src, vals, cur = {}, {}, None
for r in rows[hdr + 1:]:
    if not r:
        continue
    if r[0].isdigit():
        cur = int(r[0])
        src[cur] = r[1]
        continue
    if r[0] == "Line No":
        cur = None
        continue
    if cur is None or len(r) <= ti:
        continue
    v = r[ti].replace(",", "")
    try:
        vals[cur] = vals.get(cur, 0.0) + float(v)
    except ValueError:
        pass
name, agg = "?", {}
for ln in sorted(src):
    s = src[ln]
    if s.startswith(("__device__", "__global__", "struct")) and "(" in s and "return" not in s:
        name = s[:90]
    agg[name] = agg.get(name, 0.0) + vals.get(ln, 0.0)
tot = sum(agg.values())
print(f"total thread instructions per candidate: {tot / ncand:.0f}")
for n, v in sorted(agg.items(), key=lambda x: -x[1])[:25]:
    print(f"{100 * v / tot:5.1f}%  {v / ncand:7.0f}/cand  {n}")
