"""A GP round (bench.bench_gp's sizes) split into gp_fit and bo_propose_batch, plus the
device kernels' launch times (torch profiler-free: CUDA events around each stage)."""
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_04199_b200 import kernels as pk  # noqa: E402
from paper_2102_04199_b200 import search as ps  # noqa: E402
from paper_2102_04199_b200.util import rng_from  # noqa: E402

space = pk.build_knob_space(pk.KernelSpec(*bench.SPEC_ARGS))
rng = rng_from("bench-gp")
n, pool, batch = 512, 512, 16
obs = pk.sample_configs(space, n, rng)
x = ps.knob_coordinates(space, obs)
raw = np.sin(3.0 * x).sum(axis=1) + 0.1 * rng.normal(size=n)
y = (raw - raw.mean()) / raw.std()
pool_cfgs = pk.sample_configs(space, pool, rng)
visited = set(pk.config_index(space, c) for c in obs)
for _ in range(3):
    s = ps.gp_fit(ps.GpSurrogate(x=x, y=y, noise_variance=1e-4), select_lengthscale=True)
    ps.bo_propose_batch(s, space, batch, 2.0, pool, visited, rng_from("bench-gp-bo"), pool=pool_cfgs)
torch.cuda.synchronize()
reps = 20
tf = tb = 0.0
for _ in range(reps):
    t0 = time.perf_counter()
    s = ps.gp_fit(ps.GpSurrogate(x=x, y=y, noise_variance=1e-4), select_lengthscale=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ps.bo_propose_batch(s, space, batch, 2.0, pool, visited, rng_from("bench-gp-bo"), pool=pool_cfgs)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    tf += t1 - t0
    tb += t2 - t1
print({"gp_fit_ms": 1e3 * tf / reps, "bo_propose_ms": 1e3 * tb / reps})

if len(sys.argv) > 1 and sys.argv[1] == "--cprofile":
    import cProfile
    import pstats

    def rounds():
        for _ in range(10):
            s = ps.gp_fit(ps.GpSurrogate(x=x, y=y, noise_variance=1e-4), select_lengthscale=True)
            ps.bo_propose_batch(s, space, batch, 2.0, pool, visited, rng_from("bench-gp-bo"), pool=pool_cfgs)
        torch.cuda.synchronize()

    cProfile.run("rounds()", "/tmp/gp.prof")
    pstats.Stats("/tmp/gp.prof").sort_stats("tottime").print_stats(18)
