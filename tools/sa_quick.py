"""Time sa_explore on the device (16 chains x 128 steps, the SaSchedule defaults)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
    ps.sa_explore(pred, space, sched, set(), rng_from("sa-warm", i))
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(20):
    h = ps.sa_explore(pred, space, sched, set(), rng_from("sa-time", i))
torch.cuda.synchronize()
print(f"sa_explore (16 chains x 128 steps, device + host draws): {1e3 * (time.perf_counter() - t0) / 20:.2f} ms, "
      f"history {len(h)} configs")
