"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel total time and share.  usage: launch_summary.py launches.csv [steps]"""
import collections
import csv
import sys

path = sys.argv[1]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr, data = rows[hi], rows[hi + 1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in data:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) * {"usecond": 1e3, "msecond": 1e6}.get(r[ui], 1.0)
    name = r[ki][:80]
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
print(f"total {tot / 1e6 / steps:.3f} ms per step over {steps:g} steps, {len(data)} launches")
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
    print(f"{v / 1e6 / steps:8.3f} ms  {100 * v / tot:5.1f}%  n/step={n / steps:6.1f}  {k}")
