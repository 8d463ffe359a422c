"""Time debug variants of the tensor-core scorer (compile-time -D switches) on 1M candidates.
    python tools/tc_variants.py --build      (here)   /   python tools/tc_variants.py   (GPU box)"""
import os
import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2102_04199_b200 import build as B  # noqa: E402

VARIANTS = {"base": []}
VARIANTS.update({k: v for k, v in (a.split("=", 1) for a in sys.argv[1:] if "=" in a) for v in [v.split(",")]})


def lib_path(name):
    return ROOT / "build" / f"var_{name}" / "libkt.so"


if "--build" in sys.argv:
    for name, flags in VARIANTS.items():
        out = lib_path(name).parent
        out.mkdir(parents=True, exist_ok=True)
        objs = []
        for src in sorted(B.CSRC.glob("*.cu")):
            o = out / (src.stem + ".o")
            subprocess.run([B.nvcc(), *B.ARCH, *[f for f in B.FLAGS if f not in ("-Xptxas", "-v")], *flags,
                            "-c", str(src), "-o", str(o)], check=True)
            objs.append(str(o))
        subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", str(lib_path(name)), *objs, "-lcudart_static"],
                       check=True)
    sys.exit(0)

import torch  # noqa: E402

from paper_2102_04199_b200 import _lib  # noqa: E402

import bench  # noqa: E402
from paper_2102_04199_b200 import graphs as pg, kernels as pk, search as ps  # noqa: E402

dev = torch.device("cuda", 0)
m = None
for name in VARIANTS:
    L = _lib.load(str(lib_path(name)))
    _lib._lib = L
    if m is None:
        m = bench.bench_model(dev)
        spec = pk.KernelSpec(*bench.SPEC_ARGS)
        space = pk.build_knob_space(spec)
        lay = pg.batch_layout(spec, pg.build_super_template(pk.OP_TYPES))
        idx = torch.randint(0, space.size, (int(os.environ.get("TCV_B", 1 << 20)),), device=dev)
    for _ in range(3):
        ps.score_indices(m, spec, space, lay, idx)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        ps.score_indices(m, spec, space, lay, idx)
    e1.record()
    torch.cuda.synchronize()
    z = ps.score_indices(m, spec, space, lay, idx)
    if name == "base":
        z_base = z.clone()
    dz = (z - z_base).abs().max().item() * m.label_norm.std * 0.6931471805599453  # GFLOPS relative error
    print(f"{name:12s} {e0.elapsed_time(e1) / 20:.4f} ms per call (B={idx.numel()})   max GFLOPS rel diff vs base {dz:.2e}", flush=True)
