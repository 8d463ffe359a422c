"""Scorer / sweep paths at the bench size with a time check (regression guard for pipeline changes)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_04199_b200 import graphs as pg, kernels as pk, search as ps  # noqa: E402

m = bench.bench_model(torch.device("cuda", 0))
spec = pk.KernelSpec(*bench.SPEC_ARGS)
space = pk.build_knob_space(spec)
lay = pg.batch_layout(spec, pg.build_super_template(pk.OP_TYPES))
B = 1 << 20
idx = torch.randint(0, space.size, (B,), device="cuda")
t = time.time(); ps.score_indices(m, spec, space, lay, idx); torch.cuda.synchronize()
print("score_indices ok", time.time() - t, flush=True)
sw = ps.Sweeper(m, spec, space, lay, B, k=512)
t = time.time(); sw.run_device(idx); torch.cuda.synchronize()
print("run_device ok", time.time() - t, flush=True)
h = idx.cpu().to(torch.int32).pin_memory()
t = time.time(); sw.run_host(h); torch.cuda.synchronize()
print("run_host int32 ok", time.time() - t, flush=True)
t = time.time(); sw.run_host(idx.cpu().pin_memory()); torch.cuda.synchronize()
print("run_host int64 ok", time.time() - t, flush=True)
