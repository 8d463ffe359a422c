"""Pipeline timeline of the tensor-core scorer (CTA 0): builds a -DKT_TC_TRACE copy of
the library in build/trace/, scores 1M candidates through it, prints the per-chunk
event times (cycles, relative to the first producer arrive)."""
import ctypes
import os
import pathlib
import subprocess
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2102_04199_b200 import build as B  # noqa: E402

out = ROOT / "build" / "trace"
out.mkdir(parents=True, exist_ok=True)
lib = out / "libkt_trace.so"
if not lib.exists() or os.environ.get("REBUILD"):
    objs = []
    for src in sorted(B.CSRC.glob("*.cu")):
        o = out / (src.stem + ".o")
        extra = os.environ.get("TRACE_FLAGS", "").split()
        subprocess.run([B.nvcc(), *B.ARCH, *[f for f in B.FLAGS if f not in ("-Xptxas", "-v")], "-DKT_TC_TRACE", *extra,
                        "-c", str(src), "-o", str(o)], check=True)
        objs.append(str(o))
    subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", str(lib), *objs, "-lcudart_static"], check=True)
if "--build-only" in sys.argv:
    sys.exit(0)

import torch  # noqa: E402

from paper_2102_04199_b200 import _lib  # noqa: E402

L = _lib.load(str(lib))
L.kt_debug_trace_read.argtypes = [ctypes.c_void_p]
_lib._lib = L
import bench  # noqa: E402
from paper_2102_04199_b200 import graphs as pg, kernels as pk, search as ps  # noqa: E402

dev = torch.device("cuda", 0)
m = bench.bench_model(dev)
spec = pk.KernelSpec(*bench.SPEC_ARGS)
space = pk.build_knob_space(spec)
lay = pg.batch_layout(spec, pg.build_super_template(pk.OP_TYPES))
idx = torch.randint(0, space.size, (1 << 20,), device=dev)
for _ in range(3):
    ps.score_indices(m, spec, space, lay, idx)
torch.cuda.synchronize()
buf = np.zeros((32, 64), dtype=np.int64)
L.kt_debug_trace_read(buf.ctypes.data)
names = ["P_arrive", "G1_issued", "G2_issued", "G3_issued", "G4_issued", "E1_go", "E1_done", "E2_go", "E2_done",
         "H_u_done", "H_d3_go", "H_d4_go", "H_done"]
t0 = buf[0, 0]
print("chunk " + " ".join(f"{n:>9s}" for n in ["P_arrive", "G1_issued", "G2_issued", "E1_go", "E1_ld", "E1_rfree", "E1_st", "E1_stw", "E1_done", "E2_go", "E2_done"]))
for q in range(40):
    print(f"{q:5d} " + " ".join(f"{buf[e, q] - t0:9d}" for e in (0, 1, 2, 5, 13, 14, 15, 16, 6, 7, 8)))
print("producer tile: start v_free_ok digits_done prepared")
for ti in range(5):
    print(ti, *(buf[e, ti] - t0 for e in (24, 25, 31, 26)))
print("producer q: row_start computed x_empty_ok arrive | g1start g1commit")
for q in range(16, 40):
    print(q, buf[19, q] - t0, buf[20, q] - t0, buf[21, q] - t0, buf[0, q] - t0, "|", buf[22, q] - t0, buf[1, q] - t0)
print("G2 q: ready-seen -> last MMA issued -> committed")
for q in range(16, 40):
    print(q, buf[22, q] - t0, buf[23, q] - buf[22, q], buf[2, q] - buf[23, q])
print("MMA loop iterations 300..363: t, q2, q1")
for i in range(64):
    print(i, buf[20, i] - t0, buf[21, i] // 1000000, buf[21, i] % 1000000)
print("tile " + " ".join(f"{n:>9s}" for n in ["G3_issued", "G4_issued"] + names[9:]))
for ti in range(4):
    print(f"{ti:4d} " + " ".join(f"{buf[e, ti] - t0:9d}" for e in (3, 4, 9, 10, 11, 12)))

# single-CTA run: 55 tiles on one SM (no chip-level contention)
if "--single" in sys.argv:
    idx1 = idx[: 128 * 55].contiguous()
    for _ in range(2):
        ps.score_indices(m, spec, space, lay, idx1)
    torch.cuda.synchronize()
    L.kt_debug_trace_read(buf.ctypes.data)
    t0 = buf[0, 0]
    print("single CTA:")
    for q in range(20, 30):
        print(f"{q:5d} " + " ".join(f"{buf[e, q] - t0:9d}" for e in (0, 1, 2, 5, 6, 7, 8)))
    for ti in range(4):
        print(f"{ti:4d} " + " ".join(f"{buf[e, ti] - t0:9d}" for e in (3, 4, 9, 10, 11, 12)))
