"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, gi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0, set()])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    a = agg[r[ki][:70]]
    a[0] += 1
    a[1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)
    a[2].add(r[gi])
tot = sum(v[1] for v in agg.values())
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"total {tot / 1e3:.2f} ms over {sum(v[0] for v in agg.values())} launches")
for k, (n, t, g) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{t / 1e3:8.2f} ms {100 * t / tot:5.1f}% {n:5d} x {t / n:8.1f} us  {k}  {sorted(g)[:2]}")
