"""Single-graph API throughput (embed / forward / predict_gflops, model.py:153-169)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_04199_b200 import graphs as pg, kernels as pk, model as pm  # noqa: E402
from paper_2102_04199_b200.util import rng_from  # noqa: E402

m = bench.bench_model(torch.device("cuda", 0))
spec = pk.KernelSpec(*bench.SPEC_ARGS)
space = pk.build_knob_space(spec)
tmpl = pg.build_super_template(pk.OP_TYPES)
graphs = [pg.config_graph(spec, c, space, tmpl) for c in pk.sample_configs(space, 500, rng_from("sg"))]
for g in graphs[:20]:
    pm.predict_gflops(g, m)
t0 = time.perf_counter()
for g in graphs:
    pm.predict_gflops(g, m)
dt = time.perf_counter() - t0
print(f"predict_gflops: {len(graphs) / dt:.0f} graphs/s (first call per graph object)")
t0 = time.perf_counter()
for g in graphs:
    pm.predict_gflops(g, m)
dt = time.perf_counter() - t0
print(f"predict_gflops: {len(graphs) / dt:.0f} graphs/s (memoised tensors)")
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
for g in graphs[:200]:
    pm.predict_gflops(g, m)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
fresh = [pg.config_graph(spec, c, space, tmpl) for c in pk.sample_configs(space, 200, rng_from("sg2"))]
pr = cProfile.Profile()
pr.enable()
for g in fresh:
    pm.predict_gflops(g, m)
pr.disable()
print("--- first call per graph object")
pstats.Stats(pr).sort_stats("tottime").print_stats(16)
