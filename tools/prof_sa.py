"""Where an sa_explore call spends its time: host draws, CUDA-graph replay, history dict.

    python tools/prof_sa.py
"""
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_04199_b200 import graphs as pg  # noqa: E402
from paper_2102_04199_b200 import kernels as pk  # noqa: E402
from paper_2102_04199_b200 import search as ps  # noqa: E402
from paper_2102_04199_b200.util import rng_from  # noqa: E402

dev = torch.device("cuda", 0)
m = bench.bench_model(dev)
spec = pk.KernelSpec(*bench.SPEC_ARGS)
space = pk.build_knob_space(spec)
pred = ps.CostModelPredictor(m, spec, space, pg.batch_layout(spec, pg.build_super_template(pk.OP_TYPES)))
sched = ps.SaSchedule()
for i in range(3):
    ps.sa_explore(pred, space, sched, set(), rng_from("bench-sa-warm", i))
torch.cuda.synchronize()
reps = 20
t0 = time.perf_counter()
for i in range(reps):
    ps.sa_explore(pred, space, sched, set(), rng_from("bench-sa", i))
torch.cuda.synchronize()
total = 1e3 * (time.perf_counter() - t0) / reps
ann = next(iter(ps._ANNEALERS.values()))
n, steps, nk = ann.n, sched.steps_per_round, ann.nk
rng = rng_from("x", 0)
t0 = time.perf_counter()
for _ in range(reps):
    for s in range(steps):
        k = rng.integers(0, nk, size=n)
        rng.random(n) < 0.5
        rng.integers(0, 2, size=n) * 2 - 1
        rng.integers(0, ann.cards_np[k])
        rng.random(n)
draws = 1e3 * (time.perf_counter() - t0) / reps
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    ann._run_fused() if ann.engine == "fused" else ann.graph.replay()
e1.record()
torch.cuda.synchronize()
replay = e0.elapsed_time(e1) / reps
print({"engine": ann.engine, "total_ms": total, "python_draws_ms": draws, "device_ms": replay,
       "device_per_step_us": 1e3 * replay / steps})
