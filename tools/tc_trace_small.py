"""Latency anatomy of one scorer tile (B = 128): kernel entry, prologue, per-chunk pipeline
events, head, exit (CTA 0 clock64 stamps; needs the -DKT_TC_TRACE build of tc_trace.py)."""
import ctypes
import os
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

dev = torch.device("cuda", 0)
m = bench.bench_model(dev)
spec = pk.KernelSpec(*bench.SPEC_ARGS)
space = pk.build_knob_space(spec)
lay = pg.batch_layout(spec, pg.build_super_template(pk.OP_TYPES))
B = int(os.environ.get("B", "128"))
idx = torch.randint(0, space.size, (B,), device=dev)
for _ in range(3):
    ps.score_indices(m, spec, space, lay, idx)
torch.cuda.synchronize()
buf = np.zeros((32, 64), dtype=np.int64)
L.kt_debug_trace_read(buf.ctypes.data)
t0 = buf[27, 0]
print("entry 0  prologue_done", buf[28, 0] - t0, " exit", buf[29, 0] - t0)
print("operands", buf[30, 0] - t0, "t0 divisors", buf[30, 5] - t0, "t0 barriers", buf[30, 1] - t0,
      "tmem_alloc", buf[30, 2] - t0, "sync1", buf[30, 3] - t0, "tables", buf[30, 4] - t0)
print("chunk P_arrive G1_issued G2_issued E1_go E1_done E2_go E2_done")
for q in range(12):
    print(q, *(buf[e, q] - t0 for e in (0, 1, 2, 5, 6, 7, 8)))
print("tile G3 G4 H_u_done H_d3_go H_d4_go H_done")
print(0, *(buf[e, 0] - t0 for e in (3, 4, 9, 10, 11, 12)))
