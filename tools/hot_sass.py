"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
si, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(float(r[si] or 0) for r in data)
idx = {r[0]: i for i, r in enumerate(data)}
for r in sorted(data, key=lambda r: -float(r[si] or 0))[:n]:
    print(f"{float(r[si]) / tot * 100:5.1f}% exec={r[ei]:>8s} {r[0][-5:]} {r[1][:90]}")
