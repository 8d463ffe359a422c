"""Per-CUDA-source-line stall samples and warp-instructions from an ncu report (needs -lineinfo)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
agg = defaultdict(lambda: [0.0, 0.0, ""])
line, src = None, ""
for r in rows[hi + 1:]:
    if len(r) <= ie:
        continue
    if r[0]:
        line, src = r[0], r[1]
    try:
        agg[line][0] += float(r[si] or 0)
        agg[line][1] += float(r[ie] or 0)
        agg[line][2] = src
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"samples {tot:.0f}  warp-inst {ti:.3g}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * v[0] / tot:5.1f}% {100 * v[1] / ti:5.1f}%i L{k:>5} {v[2].strip()[:90]}")
