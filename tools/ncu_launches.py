"""Aggregate an ncu gpu__time_duration.sum launch-list CSV by kernel name (durations in us)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h, rows = rows[0], rows[1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.OrderedDict()
for r in rows:
    v = float(r[vi].replace(",", "")) * scale[r[ui]]
    a = agg.setdefault(r[ki].split("(")[0][:60], [0, 0.0])
    a[0] += 1
    a[1] += v
for n, (c, t) in agg.items():
    print(f"{n:60s} {c:4d} {t:10.1f} us {t / c:9.2f} us/launch")
print("total", sum(a[1] for a in agg.values()))
