import os, sys
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_2102_04199_b200 import graphs as pg, kernels as pk, search as ps
dev = torch.device("cuda", 0)
m = bench.bench_model(dev)
spec = pk.KernelSpec(*bench.SPEC_ARGS)
space = pk.build_knob_space(spec)
lay = pg.batch_layout(spec, pg.build_super_template(pk.OP_TYPES))
B = 1 << 20
rnd = torch.randint(0, space.size, (B,), device=dev)
base = 123456789
cont = torch.arange(base, base + B, device=dev)
z = torch.empty(B, device=dev)
def t(fn, n=300):
    for _ in range(10): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
for rep in range(2):
    print("random idx   ", round(t(lambda: ps.score_indices(m, spec, space, lay, rnd, check=False, z_out=z)), 4))
    print("contig idx   ", round(t(lambda: ps.score_indices(m, spec, space, lay, cont, check=False, z_out=z)), 4))
    print("no idx (base)", round(t(lambda: ps.score_indices(m, spec, space, lay, None, base=base, count=B, check=False, z_out=z)), 4))
