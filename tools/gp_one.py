"""One GP round at 512 observations (for profiling)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

print(bench.bench_gp(n=512, reps=2, cpu_reps=0 + 1)["value"])
