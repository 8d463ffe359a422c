"""General (non-fused) forward path at 1M graphs: encode_batch (kt_encode_raw), embed_batch through
kt_embed_csr (shared super adjacency), head_forward_batch (kt_head_forward): device ms each."""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_04199_b200 import graphs as pg, kernels as pk, model as pm  # noqa: E402
from paper_2102_04199_b200.util import rng_from  # noqa: E402

dev = torch.device("cuda", 0)
m = bench.bench_model(dev)
spec = pk.KernelSpec(*bench.SPEC_ARGS)
space = pk.build_knob_space(spec)
lay = pg.batch_layout(spec, pg.build_super_template(pk.OP_TYPES))
n = 1 << 20
idx = torch.from_numpy(rng_from("gen").integers(0, space.size, n)).to(dev)


def tm(f, reps=5):
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


feats = pg.encode_batch(spec, space, idx, lay, device=dev)
u = pm.embed_batch(m, feats, lay.feature_mask, lay.adjacency)
print({"encode_ms": tm(lambda: pg.encode_batch(spec, space, idx, lay, device=dev)),
       "embed_ms": tm(lambda: pm.embed_batch(m, feats, lay.feature_mask, lay.adjacency)),
       "head_ms": tm(lambda: pm.head_forward_batch(u, m.head))})
