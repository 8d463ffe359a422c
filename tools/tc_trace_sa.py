"""CTA-0 timeline of the fused annealing kernel (kt_sa_run, -DKT_TC_TRACE build of tc_trace.py):
per-chunk events of the first tiles and the head events per tile, cycles relative to the first
encode arrive."""
import ctypes
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2102_04199_b200 import _lib  # noqa: E402

L = _lib.load(str(ROOT / "build" / "trace" / "libkt_trace.so"))
L.kt_debug_trace_read.argtypes = [ctypes.c_void_p]
_lib._lib = L
import bench  # noqa: E402
from paper_2102_04199_b200 import graphs as pg, kernels as pk, search as ps  # noqa: E402
from paper_2102_04199_b200.util import rng_from  # noqa: E402

dev = torch.device("cuda", 0)
m = bench.bench_model(dev)
spec = pk.KernelSpec(*bench.SPEC_ARGS)
space = pk.build_knob_space(spec)
pred = ps.CostModelPredictor(m, spec, space, pg.batch_layout(spec, pg.build_super_template(pk.OP_TYPES)))
sched = ps.SaSchedule()
ann = ps.DeviceAnnealer(pred, sched, 16, engine="fused")
starts = [int(v) for v in rng_from("t", 0).integers(0, space.size, 16)]
for i in range(3):
    ann.explore(starts, rng_from("t", i))
torch.cuda.synchronize()
buf = np.zeros((32, 64), dtype=np.int64)
L.kt_debug_trace_read(buf.ctypes.data)
t0 = buf[0, 0]
ev = {"E_arr": 0, "G1_iss": 1, "R_d1": 5, "R_arr": 6, "G2_iss": 2, "O_d2": 7, "O_done": 8}
print("chunk " + " ".join(f"{k:>8s}" for k in ev))
for q in range(0, 48):
    print(f"{q:5d} " + " ".join(f"{buf[e, q] - t0:8d}" for e in ev.values()))
print("tile    G3_iss   G4_iss   H_u_arr  H_d3    H_d4    H_done  enc_top  enc_p1")
for ti in range(5):
    print(f"{ti:4d} " + " ".join(f"{buf[e, ti] - t0:8d}" for e in (3, 4, 9, 10, 11, 12, 24, 26)))
