"""GP round stage split at 512 observations: gp_fit (factor kernel, host copies) vs bo_propose_batch."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_04199_b200 import kernels as pk, search as ps  # noqa: E402
from paper_2102_04199_b200.util import rng_from  # noqa: E402

n, pool = 512, 512
space = pk.build_knob_space(pk.KernelSpec(*bench.SPEC_ARGS))
rng = rng_from("bench-gp")
obs = pk.sample_configs(space, n, rng)
x = ps.knob_coordinates(space, obs)
raw = np.sin(3.0 * x).sum(axis=1) + 0.1 * rng.normal(size=n)
y = (raw - raw.mean()) / raw.std()
pool_cfgs = pk.sample_configs(space, pool, rng)
visited = set(pk.config_index(space, c) for c in obs)


def timed(name, f, reps=10):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = f()
    torch.cuda.synchronize()
    print(f"{name:40s} {1e3 * (time.perf_counter() - t0) / reps:8.3f} ms")
    return r


s = timed("gp_fit (4 lengthscales)", lambda: ps.gp_fit(ps.GpSurrogate(x=x, y=y, noise_variance=1e-4)))
timed("gp_fit (fixed lengthscale)", lambda: ps.gp_fit(s, select_lengthscale=False))
timed("bo_propose_batch", lambda: ps.bo_propose_batch(s, space, 16, 2.0, pool, visited, rng_from("b"), pool=pool_cfgs))
L = torch.from_numpy(s.chol).cuda()
timed("chol D2H (2 MB, t().contiguous().cpu())", lambda: L.t().contiguous().cpu().numpy())
timed("knob_coordinates(pool)", lambda: ps.knob_coordinates(space, pool_cfgs))
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    ps.bo_propose_batch(s, space, 16, 2.0, pool, visited, rng_from("b"), pool=pool_cfgs)
    ps.gp_fit(ps.GpSurrogate(x=x, y=y, noise_variance=1e-4))
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
