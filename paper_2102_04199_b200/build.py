"""Build libkerntune_b200.so (all csrc/*.cu) in-tree for sm_100a with nvcc.

    python -m paper_2102_04199_b200.build [--verbose]

Objects go to build/ (git-ignored); the shared library lands next to this
file so it travels with the repo snapshot to the GPU box.  No fast-math: the
encoder's fp64 z-normalisation must stay IEEE to be bit-exact with numpy.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import pathlib
import shutil
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libkerntune_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         f"-I{ROOT / 'include'}", "-Xptxas", "-v"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _compile(src: pathlib.Path, verbose: bool) -> tuple:
    out = OBJ / (src.stem + ".o")
    deps = [src] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "kerntune_b200.h"]
    if out.exists() and all(out.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return src.name, ""
    # KT_NVCC_DEFS: extra -D switches for A/B builds of the compile-time variants
    defs = os.environ.get("KT_NVCC_DEFS", "").split()
    cmd = [nvcc(), *ARCH, *FLAGS, *defs, "-c", str(src), "-o", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
    (OBJ / (src.stem + ".ptxas.txt")).write_text(r.stderr)
    return src.name, r.stderr if verbose else ""


def build(verbose: bool = False) -> pathlib.Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu"))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for name, log in ex.map(lambda s: _compile(s, verbose), srcs):
            if log:
                print(f"--- {name}\n{log}")
    objs = [OBJ / (s.stem + ".o") for s in srcs]
    if not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs):
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart_static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    print(build(args.verbose))
    sys.exit(0)
