"""Top SASS lines by warp-stall samples from an ncu report (source page)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[hi + 1:] if len(r) > si]
tot = sum(float(r[si] or 0) for r in data)
order = sorted(range(len(data)), key=lambda i: -float(data[i][si] or 0))
for i in sorted(order[:n]):
    r = data[i]
    print(f"{i:5d} {float(r[si] or 0) / tot * 100:5.1f}%  {r[1][:90]}")
