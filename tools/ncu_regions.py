"""Thread instructions and stall samples per source-line range of engine.cu (ncu source page CSV).

    python tools/ncu_regions.py src.csv n_candidates name:lo-hi [name:lo-hi ...]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
ncand = float(sys.argv[2])
ranges = []
for a in sys.argv[3:]:
    name, r = a.split(":")
    lo, hi = map(int, r.split("-"))
    ranges.append((name, lo, hi))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr]
ti = h.index("Thread Instructions Executed")
si = h.index("Warp Stall Sampling (All Samples)")
agg = {n: [0.0, 0.0] for n, _, _ in ranges}
agg["other"] = [0.0, 0.0]
cur = None
for r in rows[hdr + 1:]:
    if len(r) < len(h):
        continue
    if r[0]:
        cur = int(r[0]) if r[0].isdigit() else None
        if cur is None:
            continue
        name = next((n for n, lo, hi in ranges if lo <= cur <= hi), "other")
        for j, c in ((0, ti), (1, si)):
            try:
                agg[name][j] += float(r[c].replace(",", ""))
            except ValueError:
                pass
tot = [sum(v[j] for v in agg.values()) for j in (0, 1)]
print(f"thread instructions per candidate: {tot[0] / ncand:.0f}")
for n, v in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{n:16s} instr {v[0] / ncand:7.0f}/cand ({100 * v[0] / tot[0]:5.1f}%)  stalls {100 * v[1] / max(tot[1], 1):5.1f}%")
