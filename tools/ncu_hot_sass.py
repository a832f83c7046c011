"""Top SASS lines by warp-stall samples from an .ncu-rep (source page):
python tools/ncu_hot_sass.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
ia, isrc, ist = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[2:] if len(r) > ist]
tot = sum(float(r[ist] or 0) for r in data)
idx = {r[ia]: i for i, r in enumerate(data)}
for r in sorted(data, key=lambda r: -float(r[ist] or 0))[:n]:
    i = idx[r[ia]]
    prev = data[i - 1][isrc].strip() if i > 0 else ""
    print(f"{float(r[ist]) / tot * 100:5.1f}%  {r[isrc].strip()[:70]:70s} | prev: {prev[:50]}")
