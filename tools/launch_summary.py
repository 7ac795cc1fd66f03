"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel name,
count, total and mean device time, and share of the listed time (our kernels and torch's)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0}
for r in rows[1:]:
    name = r[ki].split("(")[0]
    us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)
    c, t = agg.get(name, (0, 0.0))
    agg[name] = (c + 1, t + us)
mine = {k: v for k, v in agg.items() if "sb::" in k}
tot = sum(t for _, t in mine.values())
print(f"{'kernel':45s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
for k, (c, t) in sorted(mine.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:45]:45s} {c:8d} {t:10.1f} {t / c:9.1f} {100 * t / tot:5.1f}%")
other = sum(t for k, (c, t) in agg.items() if k not in mine)
print(f"(other kernels in the process, e.g. input generation: {other:.1f} us)")
