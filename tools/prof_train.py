"""Launch a few of each secondary-path step (C2 grad + SGD at batch 512, C3 MAML FO / SO,
C4 fine-tune, the streaming aggregation kernels) for an ncu launch list:

    ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_train.py
"""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_04199_b200 import meta as pmeta  # noqa: E402
from paper_2102_04199_b200 import model as pm  # noqa: E402

dev = torch.device("cuda", 0)
m = bench.bench_model(dev)
entries = bench.synthetic_entries()
corpus = bench.synthetic_corpus(entries)
fn, ln = pmeta.dataset_norms(corpus)
m = pm.model_from_flat(m._flat, m, feature_norm=fn, label_norm=ln)
what = sys.argv[1:] or ["pretrain", "maml", "fine_tune", "aggregate"]
N = int(__import__("os").environ.get("PROF_STEPS", "5"))  # timed steps (more for A/B timing runs)
if "pretrain" in what:
    print(bench.bench_pretrain_step(m, bench.synthetic_corpus(entries, ("conv2d", "winograd", "depthwise")), N, 3))
if "maml" in what:
    print(bench.bench_maml(m, corpus, N, 3))
    print(bench.bench_maml(m, corpus, N, 3, first_order=False))
if "fine_tune" in what:
    print(bench.bench_fine_tune(m, corpus, reps=N))
if "aggregate" in what:
    print(bench.bench_aggregate(m, reps=2))
torch.cuda.synchronize()
