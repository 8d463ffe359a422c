"""Top-k of the sweep step alone: kt_topk_keys on the keys of one scored 1M batch (first-digit bins
counted by the top-k itself, hist_ready = 0), and the scorer + top-k pair as the bench runs it."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_04199_b200 import _lib, graphs as pg, kernels as pk, search as ps  # noqa: E402

dev = torch.device("cuda", 0)
m = bench.bench_model(dev)
spec = pk.KernelSpec(*bench.SPEC_ARGS)
space = pk.build_knob_space(spec)
lay = pg.batch_layout(spec, pg.build_super_template(pk.OP_TYPES))
B = 1 << 20
idx = torch.randint(0, space.size, (B,), device=dev)
sw = ps.Sweeper(m, spec, space, lay, B, k=512)
st = _lib.stream_handle()
p = sw._p


def timed(fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1000.0


sw.score(idx.data_ptr(), None, 0, B, st)
torch.cuda.synchronize()
topk_alone = timed(lambda: _lib.check(sw.lib.kt_topk_keys(p["keys"], B, sw.k, 0, p["ti"], p["ts"], p["ws"],
                                                          sw.ws_bytes, st), "topk"))
score_alone = timed(lambda: sw.score(idx.data_ptr(), None, 0, B, st))
pair = timed(lambda: (sw.score(idx.data_ptr(), None, 0, B, st), sw.rank(B, st)))
print({"topk_keys_us (own first pass)": round(topk_alone, 2), "score_us": round(score_alone, 2),
       "score+rank_us": round(pair, 2), "rank_in_pair_us": round(pair - score_alone, 2)})
