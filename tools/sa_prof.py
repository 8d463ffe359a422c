"""Break sa_explore's wall time into host draws, graph replay and history building."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_04199_b200 import graphs as pg, kernels as pk, search as ps  # noqa: E402
from paper_2102_04199_b200.util import rng_from  # noqa: E402

m = bench.bench_model(torch.device("cuda", 0))
spec = pk.KernelSpec(*bench.SPEC_ARGS)
space = pk.build_knob_space(spec)
pred = ps.CostModelPredictor(m, spec, space, pg.batch_layout(spec, pg.build_super_template(pk.OP_TYPES)))
sched = ps.SaSchedule()
for i in range(3):
    ps.sa_explore(pred, space, sched, set(), rng_from("w", i))
ann = next(iter(ps._ANNEALERS.values()))
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(20):
    ps.sa_explore(pred, space, sched, set(), rng_from("x", i))
torch.cuda.synchronize()
print("sa_explore ms", 1e3 * (time.perf_counter() - t0) / 20)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(20):
    ann.graph.replay()
e1.record()
torch.cuda.synchronize()
print("graph replay ms", e0.elapsed_time(e1) / 20)
rng = rng_from("d")
t0 = time.perf_counter()
for i in range(20):
    for s in range(128):
        k = rng.integers(0, 8, size=16)
        rng.random(16) < 0.5
        rng.integers(0, 2, size=16) * 2 - 1
        rng.integers(0, ann.cards_np[k])
        rng.random(16)
print("host draws ms", 1e3 * (time.perf_counter() - t0) / 20)
