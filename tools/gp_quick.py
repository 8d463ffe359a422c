"""GP round bench only (bench.bench_gp) on cuda:0; prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

for n in (64, 256, 512):
    print(json.dumps(bench.bench_gp(n=n)))
