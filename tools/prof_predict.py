"""C1 predict split: configs_to_indices vs the device call vs the whole CostModelPredictor call."""
import sys, time, pathlib
ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np, torch
import bench
from paper_2102_04199_b200 import graphs as pg, kernels as pk, search as ps
from paper_2102_04199_b200.util import rng_from
dev = torch.device("cuda", 0)
m = bench.bench_model(dev)
spec = pk.KernelSpec(*bench.SPEC_ARGS); space = pk.build_knob_space(spec)
lay = pg.batch_layout(spec, pg.build_super_template(pk.OP_TYPES))
pred = ps.CostModelPredictor(m, spec, space, lay)
cf = pk.sample_configs(space, 4096, rng_from("pp"))
for _ in range(5): pred(cf)
torch.cuda.synchronize()
N=200
t0=time.perf_counter()
for _ in range(N): pg.configs_to_indices(space, cf)
t1=time.perf_counter()
idx = pg.configs_to_indices(space, cf)
for _ in range(N): pred._fast(idx, False)
t2=time.perf_counter()
for _ in range(N): pred(cf)
t3=time.perf_counter()
print({"c2i_us": 1e6*(t1-t0)/N, "fast_us": 1e6*(t2-t1)/N, "call_us": 1e6*(t3-t2)/N})
