"""Summarise an ncu source page (cuda,sass CSV) by CUDA source line: stall samples and executed instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr]
ci = {n: h.index(n) for n in ("Warp Stall Sampling (All Samples)", "Instructions Executed",
                               "Thread Instructions Executed")}
lines, cur = {}, None
for r in rows[hdr + 1:]:
    if len(r) < len(h):
        continue
    if r[0]:
        if not r[0].isdigit():
            cur = None
            continue
        cur = (int(r[0]), r[1][:90])
        lines.setdefault(cur, [0, 0, 0])
        continue
    if cur is None:
        continue
    acc = lines[cur]
    for j, n in enumerate(ci):
        v = r[ci[n]].replace(",", "")
        acc[j] += float(v) if v not in ("", "-") else 0.0
tot = [sum(v[j] for v in lines.values()) for j in range(3)]
print(f"total stall samples {tot[0]:.0f}, warp instrs {tot[1]:.3e}, thread instrs {tot[2]:.3e}")
key = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for (ln, src), v in sorted(lines.items(), key=lambda kv: -kv[1][key])[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{ln:5d} stall {100*v[0]/max(tot[0],1):5.1f}%  instr {100*v[1]/max(tot[1],1):5.1f}%  "
          f"thr/instr {v[2]/max(v[1],1):5.1f}  {src}")
