"""Stall-reason breakdown per CUDA source line range from an ncu report (needs -lineinfo).
    python tools/ncu_stalls.py REPORT FILE_SUBSTR LO-HI [LO-HI ...]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, fsub = sys.argv[1], sys.argv[2]
ranges = [tuple(map(int, a.split("-"))) for a in sys.argv[3:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
st = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
ie = h.index("Instructions Executed")
line = None
acc = {rg: defaultdict(float) for rg in ranges}
for r in rows[hi + 1:]:
    if len(r) <= ie:
        continue
    if r[0]:
        try:
            line = int(r[0])
        except ValueError:
            line = None
    if line is None:
        continue
    for rg in ranges:
        if rg[0] <= line <= rg[1]:
            for i in st:
                try:
                    acc[rg][h[i]] += float(r[i] or 0)
                except ValueError:
                    pass
            try:
                acc[rg]["inst"] += float(r[ie] or 0)
            except ValueError:
                pass
for rg in ranges:
    a = acc[rg]
    tot = sum(v for k, v in a.items() if k != "inst") or 1
    top = sorted(((v, k) for k, v in a.items() if k != "inst"), reverse=True)[:8]
    print(f"lines {rg[0]}-{rg[1]}: samples {tot:.0f}, warp-inst {a['inst']:.3g}: " +
          ", ".join(f"{k[6:]} {100 * v / tot:.0f}%" for v, k in top))
