"""Small driver for ncu: one fine-tune call, a few MAML steps, one pretrain step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2102_04199_b200 import meta as pmeta
from paper_2102_04199_b200 import model as pm

dev = torch.device("cuda", 0)
m = bench.bench_model(dev)
corpus = bench.synthetic_corpus(bench.synthetic_entries(n_kernels=8, per_kernel=64))
fn, ln = pmeta.dataset_norms(corpus)
m = pm.model_from_flat(m._flat, m, feature_norm=fn, label_norm=ln)
print(bench.bench_fine_tune(m, corpus, reps=3))
print(bench.bench_maml(m, corpus, 5, 3))
print(bench.bench_pretrain_step(m, corpus, 3, 3))
