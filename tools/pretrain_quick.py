"""C2 pretrain-step bench only (bench.bench_pretrain_step) on cuda:0; prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_04199_b200 import meta as pmeta  # noqa: E402
from paper_2102_04199_b200 import model as pm  # noqa: E402

dev = torch.device("cuda", 0)
m = bench.bench_model(dev)
entries = bench.synthetic_entries()
corpus = bench.synthetic_corpus(entries, ("conv2d", "winograd", "depthwise"))
fn, ln = pmeta.dataset_norms(corpus)
m = pm.model_from_flat(m._flat, m, feature_norm=fn, label_norm=ln)
print(json.dumps(bench.bench_pretrain_step(m, corpus, int(os.environ.get("STEPS", "50")), 5)))
