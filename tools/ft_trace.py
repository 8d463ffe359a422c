"""Phase timeline of the fine-tune cluster kernel (CTA 0; -DKT_META_TRACE build in build/alt/mtrace.so):
clock64 after the head pass's barriers and around the two cluster barriers of every step."""
import ctypes
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2102_04199_b200 import _lib  # noqa: E402

L = _lib.load(str(ROOT / "build" / "alt" / "mtrace.so"))
L.kt_meta_trace_read.argtypes = [ctypes.c_void_p]
_lib._lib = L
import bench  # noqa: E402
from paper_2102_04199_b200 import meta as pmeta, model as pm  # noqa: E402

dev = torch.device("cuda", 0)
m = bench.bench_model(dev)
corpus = bench.synthetic_corpus(bench.synthetic_entries())
fn, ln = pmeta.dataset_norms(corpus)
m = pm.model_from_flat(m._flat, m, feature_norm=fn, label_norm=ln)
print(bench.bench_fine_tune(m, corpus, reps=1))
torch.cuda.synchronize()
buf = np.zeros(512, dtype=np.int64)
L.kt_meta_trace_read(buf.ctypes.data)
ev = buf.reshape(-1, 2)
t0 = ev[0, 1]
prev = t0
for line, t in ev[:60]:
    if line == 0:
        break
    print(f"line {line:5d}  +{t - prev:6d}  @{t - t0:7d}")
    prev = t
