"""Time head-engine variants (fine-tune C4, MAML C3 step) built with different -D switches.
    python tools/meta_variants.py --build NAME=-DFLAG,...   (here)   /   python tools/meta_variants.py NAME=... (GPU box)"""
import os
import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2102_04199_b200 import build as B  # noqa: E402

VARIANTS = {"base": []}
VARIANTS.update({k: v.split(",") for k, v in (a.split("=", 1) for a in sys.argv[1:] if "=" in a)})


def lib_path(name):
    return ROOT / "build" / f"mvar_{name}" / "libkt.so"


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

import bench  # noqa: E402
from paper_2102_04199_b200 import _lib  # noqa: E402
from paper_2102_04199_b200 import meta as pmeta  # noqa: E402
from paper_2102_04199_b200 import model as pm  # noqa: E402

dev = torch.device("cuda", 0)
base_m = None
for name in VARIANTS:
    _lib._lib = _lib.load(str(lib_path(name)))
    if base_m is None:
        base_m = bench.bench_model(dev)
        entries = bench.synthetic_entries(n_kernels=12, per_kernel=64)
        corpus = bench.synthetic_corpus(entries)
        fn, ln = pmeta.dataset_norms(corpus)
        m = pm.model_from_flat(base_m._flat, base_m, feature_norm=fn, label_norm=ln)
    ft = bench.bench_fine_tune(m, corpus)
    ml = bench.bench_maml(m, corpus, 100, 10)
    print(f"{name:10s} fine-tune {ft['value']:.4f} ms   maml {ml['ms_per_step'] * 1e3:.1f} us/step", flush=True)
