"""Top SASS instructions by warp-stall samples with the dominant stall reasons (ncu source page)."""
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
st = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[si] or 0) for r in data)
for idx, r in sorted(enumerate(data), key=lambda x: -float(x[1][si] or 0))[:n]:
    reasons = sorted(((float(r[i] or 0), h[i][6:]) for i in st), reverse=True)[:3]
    rs = " ".join(f"{nm}:{v:.0f}" for v, nm in reasons if v > 0)
    prev = data[idx - 1][1][:40] if idx > 0 else ""
    print(f"{float(r[si]) / tot * 100:5.1f}% exec={r[ei]:>8s} {r[1][:50]:50s} | {rs} | prev: {prev}")
