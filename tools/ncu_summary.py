"""Summarise an ncu --set full report: headline metrics, stall reasons, SASS opcode mix."""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
if len(r) >= 3:
    units, v = r[1], r[2]
else:
    units, v = [''] * len(h), r[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]
out = {}
for w in want:
    if w in h:
        i = h.index(w)
        out[w] = (v[i], units[i])
        print(f"{w:70s} {v[i]} {units[i]}")
print("-- stalls per issue")
st = []
for i, n in enumerate(h):
    if "warps_issue_stalled" in n and n.endswith("per_issue_active.ratio"):
        try:
            st.append((float(v[i]), n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
for val, n in sorted(st, reverse=True)[:10]:
    print(f"  {n:30s} {val:.3f}")
if "--sass" in sys.argv:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hh = rows[1]
    si, so, ie = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source"), hh.index("Instructions Executed")
    c, ci = Counter(), Counter()
    tot = 0
    for row in rows[2:]:
        if len(row) <= si or not row[si]:
            continue
        toks = row[so].split()
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        c[op] += float(row[si]); ci[op] += float(row[ie] or 0); tot += float(row[si])
    print("-- SASS opcode share of stall samples (and warp-instructions executed)")
    for op, val in c.most_common(18):
        print(f"  {op:10s} {100 * val / tot:5.1f}%  {ci[op]:.3g}")
