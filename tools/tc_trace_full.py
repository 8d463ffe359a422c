"""Full per-chunk pipeline timeline of the tensor-core scorer (CTA 0, -DKT_TC_TRACE build in
build/trace/, see tc_trace.py): every stamped event for chunks LO..HI, cycles relative to
the first encode arrive, plus the head events per tile."""
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

dev = torch.device("cuda", 0)
m = bench.bench_model(dev)
spec = pk.KernelSpec(*bench.SPEC_ARGS)
space = pk.build_knob_space(spec)
lay = pg.batch_layout(spec, pg.build_super_template(pk.OP_TYPES))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
idx = torch.randint(0, space.size, (n,), device=dev)
for _ in range(3):
    ps.score_indices(m, spec, space, lay, idx)
torch.cuda.synchronize()
buf = np.zeros((32, 64), dtype=np.int64)
L.kt_debug_trace_read(buf.ctypes.data)
t0 = buf[0, 0]
ev = {"E_row": 19, "E_xwait": 20, "E_xok": 21, "E_arr": 0, "G1_wait": 22, "G1_ok": 23, "G1_iss": 1,
      "R_d1": 5, "R_ld": 13, "R_rfree": 14, "R_st": 15, "R_stw": 16, "R_arr": 6, "G2_wait": 17, "G2_ok": 18,
      "G2_iss": 2, "O_d2": 7, "O_done": 8}
print("chunk " + " ".join(f"{k:>8s}" for k in ev))
for q in range(0, 64):
    print(f"{q:5d} " + " ".join(f"{buf[e, q] - t0:8d}" for e in ev.values()))
print("tile    G3_iss   G4_iss   H_u_arr  H_d3    H_d4    H_done")
for ti in range(6):
    print(f"{ti:4d} " + " ".join(f"{buf[e, ti] - t0:8d}" for e in (3, 4, 9, 10, 11, 12)))
print("encode tile: top  ok  phase1_start  first_row")
for ti in range(6):
    print(ti, buf[24, ti] - t0, buf[25, ti] - t0, buf[26, ti] - t0, buf[19, ti * 12] - t0)
print("kernel entry / prologue / exit:", buf[27, 0] - t0, buf[28, 0] - t0, buf[29, 0] - t0)
