"""Markdown table of every kernel in an ncu --set full report (the profiles/ summaries):
time, DRAM bytes, throughput, issue / warp activity, launch shape, bank conflicts, top stalls.

    python tools/ncu_table.py report.ncu-rep [time unit: us|ms]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
unit = sys.argv[2] if len(sys.argv) > 2 else "us"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
cols = [("gpu__time_duration.sum", "time " + unit), ("dram__bytes_read.sum", "DRAM read MB"),
        ("dram__bytes_write.sum", "DRAM write MB"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"), ("launch__grid_size", "grid"),
        ("launch__block_size", "block"), ("launch__registers_per_thread", "regs"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld conflicts")]


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


units = rows[1]
print("| kernel | " + " | ".join(c[1] for c in cols) + " | top stalls (per issue) |")
print("|---|" + "---|" * (len(cols) + 1))
for v in rows[2:]:
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    cells = []
    for k, _ in cols:
        x = num(d.get(k, ""))
        if x is None:
            cells.append("")
            continue
        if k == "gpu__time_duration.sum":  # report in the requested unit
            scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3}.get(u[k], 1.0)
            x = x * scale / (1e3 if unit == "ms" else 1.0)
        if k.startswith("dram__bytes"):
            scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u[k], 1.0)
            x *= scale
        cells.append(f"{x:.3f}" if x < 1000 else f"{x:.0f}")
    st = sorted(((num(d[k]) or 0.0, k) for k in h if k.startswith("smsp__average_warps_issue_stalled_")
                 and k.endswith("_per_issue_active.ratio") and num(d[k]) is not None), reverse=True)[:4]
    stalls = ", ".join(f"{k[34:-23]} {x:.2f}" for x, k in st)
    name = d["Kernel Name"].split("(")[0].replace("kt::", "")
    print(f"| `{name}` | " + " | ".join(cells) + f" | {stalls} |")
