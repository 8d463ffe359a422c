"""Race guard for the fused annealer: many explores with fresh seeds, each history compared with the
per-step kernels' (any mismatch or hang would show a handshake race in kt_sa_run)."""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_04199_b200 import graphs as pg, kernels as pk, search as ps  # noqa: E402
from paper_2102_04199_b200.util import rng_from  # noqa: E402

dev = torch.device("cuda", 0)
m = bench.bench_model(dev)
spec = pk.KernelSpec(*bench.SPEC_ARGS)
space = pk.build_knob_space(spec)
pred = ps.CostModelPredictor(m, spec, space, pg.batch_layout(spec, pg.build_super_template(pk.OP_TYPES)))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
bad = 0
for chains in (16, 128, 37):
    sched = ps.SaSchedule(steps_per_round=64, parallel_chains=chains)
    fused = ps.DeviceAnnealer(pred, sched, chains, engine="fused")
    steps = ps.DeviceAnnealer(pred, sched, chains, engine="steps")
    for i in range(n):
        starts = [int(v) for v in rng_from("race-starts", chains, i).integers(0, space.size, chains)]
        a = fused.explore(starts, rng_from("race", chains, i))
        b = steps.explore(starts, rng_from("race", chains, i))
        bad += list(a.items()) != list(b.items())
print({"explores": 3 * n, "mismatches": bad})
