"""Aggregation-kernel bench only (bench.bench_aggregate) on cuda:0; prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

m = bench.bench_model(torch.device("cuda", 0))
print(json.dumps(bench.bench_aggregate(m), indent=1))
