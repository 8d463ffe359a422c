"""sa_explore call time (bench_sa) alone: PDL on vs KT_NO_PDL=1 A/B."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

m = bench.bench_model(torch.device("cuda", 0))
print(os.environ.get("KT_NO_PDL", "pdl"), bench.bench_sa(m))
