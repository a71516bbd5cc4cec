"""Top CUDA source lines by one warp-stall reason (ncu source page CSV with per-reason columns).

    python tools/ncu_stalls.py src.csv [reason ...]     e.g. stall_short_sb stall_long_sb
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr]
for reason in sys.argv[2:] or ["stall_short_sb", "stall_long_sb"]:
    c = h.index(reason)
    out = []
    for r in rows[hdr + 1:]:
        if len(r) < len(h) or not r[0].isdigit():
            continue
        try:
            out.append((float(r[c].replace(",", "")), int(r[0]), r[1][:100]))
        except ValueError:
            pass
    tot = sum(x[0] for x in out) or 1
    print(f"== {reason} (total {tot:.0f})")
    for v, ln, src in sorted(out, reverse=True)[:12]:
        print(f"{100 * v / tot:5.1f}% {ln:5d} {src}")
