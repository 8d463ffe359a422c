"""Kernel-only time of the tensor-core scorer at small batch sizes (fixed-cost check)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_04199_b200 import _lib, graphs as pg, kernels as pk  # noqa: E402
from paper_2102_04199_b200.model import dims_of, flat_params  # noqa: E402

dev = torch.device("cuda", 0)
m = bench.bench_model(dev)
spec = pk.KernelSpec(*bench.SPEC_ARGS)
space = pk.build_knob_space(spec)
lay = pg.batch_layout(spec, pg.build_super_template(pk.OP_TYPES))
tab = pg.device_spec_table(spec, space, lay, m.feature_norm.mean, m.feature_norm.std, device=dev)
lib = _lib.load()
flat, d = flat_params(m), dims_of(m)
err = torch.zeros(1, dtype=torch.int32, device=dev)
st = _lib.stream_handle()
for B in (16, 128, 1024, 18944, 1 << 20):
    idx = torch.randint(0, space.size, (B,), device=dev)
    z = torch.empty(B, device=dev)
    fn = lib.kt_score_indices_fp32 if os.environ.get("ENGINE") == "fp32" else lib.kt_score_indices
    f = lambda: fn(tab.data_ptr(), d, flat.data_ptr(), idx.data_ptr(), 0, B, z.data_ptr(), None,
                                     err.data_ptr(), st)
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        f()
    e1.record()
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    for _ in range(50):
        f()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"B={B:8d}  {1e3 * e0.elapsed_time(e1) / 50:9.1f} us per launch  host us {(t1 - t0) / 50 * 1e6:.1f}")
