import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2102_04199_b200 import meta as pmeta, model as pm
from paper_2102_04199_b200.util import rng_from
dev = torch.device("cuda", 0)
m = bench.bench_model(dev)
corpus = bench.synthetic_corpus()
cfg = pmeta.MetaConfig(n_way=3, k_shot=2, meta_batch=32)
tr = pmeta.MetaTrainer(m, corpus, cfg)
plan = tr.plan(rng_from("metatrain", "super", 0), 30)
bufs = tr._buffers(plan)
for s in range(30):
    tr.step(plan, bufs, s)
    torch.cuda.synchronize()
    st = bufs["stats"][s].cpu().numpy()
    th = pm.flat_params(tr.model())
    print(s, st / 32, float(th.abs().max()), bool(torch.isfinite(bufs["u"]).all()), float(bufs["u"].abs().max()),
          bool(torch.isfinite(bufs["g"]).all()), float(plan["y"][s].abs().max()))
    if not np.isfinite(st).all():
        break
u, y = pmeta._embedded(m, corpus[:64])
print("embedded finite", bool(torch.isfinite(u).all()), float(u.abs().max()))
fn = m.feature_norm
print("fnorm", fn.mean, fn.std)
