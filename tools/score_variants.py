"""A/B variants of the tensor-core scorer: build copies of the library with extra -D flags
(here, CPU) and time kt_score_indices on 1M conv2d candidates with each (GPU box).

    python tools/score_variants.py build NAME="-DFOO=1" NAME2="-DBAR=2" ...
    python tools/score_variants.py run            # times every built variant + the product lib
"""
import os
import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
OUT = ROOT / "build" / "variants"


def build(specs):
    from paper_2102_04199_b200 import build as B

    OUT.mkdir(parents=True, exist_ok=True)
    base_objs = [B.OBJ / (s.stem + ".o") for s in sorted(B.CSRC.glob("*.cu")) if s.stem != "kt_score_tc"]
    B.build()
    for spec in specs:
        name, flags = spec.split("=", 1)
        o = OUT / f"kt_score_tc_{name}.o"
        subprocess.run([B.nvcc(), *B.ARCH, *[f for f in B.FLAGS if f not in ("-Xptxas", "-v")], *flags.split(),
                        "-c", str(B.CSRC / "kt_score_tc.cu"), "-o", str(o)], check=True)
        subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", str(OUT / f"lib_{name}.so"), str(o),
                        *map(str, base_objs), "-lcudart_static"], check=True)
        print("built", name, flags)


def run():
    import torch

    from paper_2102_04199_b200 import _lib

    libs = [("product", None)] + [(p.stem[4:], str(p)) for p in sorted(OUT.glob("lib_*.so"))]
    import bench
    from paper_2102_04199_b200 import graphs as pg, kernels as pk, search as ps

    dev = torch.device("cuda", 0)
    res = {}
    for rnd in range(2):
        for name, path in libs:
            _lib._lib = None
            L = _lib.load(path) if path else _lib.load()
            _lib._lib = L
            m = bench.bench_model(dev)
            spec = pk.KernelSpec(*bench.SPEC_ARGS)
            space = pk.build_knob_space(spec)
            lay = pg.batch_layout(spec, pg.build_super_template(pk.OP_TYPES))
            idx = torch.randint(0, space.size, (1 << 20,), device=dev, generator=torch.Generator(dev).manual_seed(1))
            z0 = ps.score_indices(m, spec, space, lay, idx)
            for _ in range(5):
                ps.score_indices(m, spec, space, lay, idx, z_out=z0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(50):
                ps.score_indices(m, spec, space, lay, idx, z_out=z0, check=False)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 50
            res.setdefault(name, []).append(ms)
            if rnd == 1:
                zr = res.setdefault("_z", {})
                zr[name] = z0.clone()
    zref = res["_z"]["product"]
    for name, _ in libs:
        same = torch.equal(res["_z"][name], zref)
        print(f"{name:24s} {min(res[name]):.4f} ms  {res[name]}  identical_scores={same}")


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        run()
