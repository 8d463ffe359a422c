"""meta.pretrain (batch-1 SGD epochs, meta.py:104-123) throughput on the 47 x 200 corpus."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_04199_b200 import meta as pmeta  # noqa: E402
from paper_2102_04199_b200.util import rng_from  # noqa: E402

corpus = bench.synthetic_corpus(bench.synthetic_entries())
cfg = pmeta.MetaConfig(pretrain_epochs=1, gamma=0.005)
pmeta.pretrain(corpus, cfg, rng_from("pe", 0))
torch.cuda.synchronize()
for epochs in (1, 3):
    cfg = pmeta.MetaConfig(pretrain_epochs=epochs, gamma=0.005)
    t0 = time.perf_counter()
    pmeta.pretrain(corpus, cfg, rng_from("pe", epochs))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"epochs {epochs}: {dt:.3f} s  {epochs * len(corpus) / dt:.0f} samples/s")
