"""C4 fine-tune + C3 MAML timings only (bench.bench_fine_tune / bench_maml) on cuda:0."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_04199_b200 import meta as pmeta  # noqa: E402
from paper_2102_04199_b200 import model as pm  # noqa: E402

dev = torch.device("cuda", 0)
m = bench.bench_model(dev)
corpus = bench.synthetic_corpus(bench.synthetic_entries(n_kernels=12, per_kernel=64))
fn, ln = pmeta.dataset_norms(corpus)
m = pm.model_from_flat(m._flat, m, feature_norm=fn, label_norm=ln)
print("fine-tune ms/call", bench.bench_fine_tune(m, corpus)["value"])
print("maml us/step", 1e3 * bench.bench_maml(m, corpus, 100, 10)["ms_per_step"])
