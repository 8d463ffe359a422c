"""Multi-rank execution of the device path: two processes on cuda:0 over
gloo (device tensors staged through the host by dist.py; the same code runs NCCL on a
multi-GPU node), the real sm_100a kernels on every rank.

  * candidate sweep: Sweeper on each rank's contiguous half of 2M candidates + the
    all-gathered top-k merge == one rank's Sweeper over all 2M, bit for bit;
  * MAML: MetaTrainer(shard=(rank, 2)) theta after 20 outer steps (FO) / 6 (SO) ==
    the one-rank MetaTrainer, bit for bit (per-task rows all-gathered, summed in task
    order: meta.py:223-257 "sum, not mean"); dist.meta_step_dp == meta.meta_step bit for bit;
  * grad: dist.grad_dp == model.grad within rel 1e-6 (batch-mean all-reduce).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world_size, port, results):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    out = {}
    try:
        from paper_2102_04199_b200 import dist as pd
        from paper_2102_04199_b200 import graphs as pg
        from paper_2102_04199_b200 import kernels as pk
        from paper_2102_04199_b200 import meta as pmeta
        from paper_2102_04199_b200 import model as pm
        from paper_2102_04199_b200 import search as ps
        from paper_2102_04199_b200.util import rng_from
        from tests._shared import device_model
        from tests.conftest import load_golden
        from tests.test_gpu_train import corpus_samples

        dev = torch.device("cuda", 0)
        # 1) sweep
        m = device_model(load_golden("baseline"), device=dev)
        spec = pk.KernelSpec("conv2d", 56, 64, 64, 3, 3, 1)
        space = pk.build_knob_space(spec)
        lay = pg.batch_layout(spec, pg.build_super_template(pk.OP_TYPES))
        n = 2 << 20
        idx = torch.from_numpy(rng_from("dist-sweep").integers(0, space.size, n)).to(dev)
        lo, hi = pd.shard_bounds(n, rank, world_size)
        sw = ps.Sweeper(m, spec, space, lay, hi - lo, k=512)
        ti, ts = sw.run_device(idx[lo:hi])
        gi, gs = pd.allgather_topk(ti.clone(), ts.clone(), 512)
        one = ps.Sweeper(m, spec, space, lay, n, k=512)
        ri, rs = one.run_device(idx)
        out["sweep"] = bool(torch.equal(gi, ri) and torch.equal(gs, rs))

        # 2) MAML: MetaTrainer and meta_step_dp, one rank vs two
        g_model, g_meta, g_enc = load_golden("model"), load_golden("meta"), load_golden("encode")
        m = device_model(g_model, device=dev)
        samples = corpus_samples(g_enc, g_meta, True)
        for order, fo, steps in (("fo", True, 20), ("so", False, 6)):
            cfg = pmeta.MetaConfig(n_way=3, k_shot=2, meta_batch=32, inner_steps=1, first_order=fo)
            solo = pmeta.MetaTrainer(m, samples, cfg)
            plan1 = solo.plan(rng_from("dist-maml", order), steps)
            b1 = solo.run(plan1)
            dp = pmeta.MetaTrainer(m, samples, cfg)
            plan2 = dp.plan(rng_from("dist-maml", order), steps, shard=(rank, world_size))
            b2 = dp.run(plan2)
            torch.cuda.synchronize()
            out[f"trainer_{order}"] = bool(torch.equal(pm.flat_params(dp.model()), pm.flat_params(solo.model())))
            out[f"trainer_{order}_stats"] = bool(np.array_equal(dp.stats(plan2, b2), solo.stats(plan1, b1)))
        cfg = pmeta.MetaConfig(n_way=3, k_shot=2, meta_batch=32, inner_steps=1, first_order=True)
        tasks = pmeta.sample_meta_tasks(samples, cfg, rng_from("dist-meta-step"))
        m1, st1 = pmeta.meta_step(m, tasks, cfg)
        m2, st2 = pd.meta_step_dp(m, tasks, cfg)
        d12 = (pm.flat_params(m1) - pm.flat_params(m2)).abs()
        out["meta_step_dp"] = bool(torch.equal(pm.flat_params(m1), pm.flat_params(m2))) or \
            f"max |diff| {float(d12.max()):.3e} at {int(d12.argmax())} of {d12.numel()}"
        out["meta_step_dp_stats"] = abs(st1["query_loss"] - st2["query_loss"]) <= 1e-12 * abs(st1["query_loss"])

        # 3) grad: data parallel batch mean vs one rank
        batch = [(s.graph, s.label_gflops) for s in samples[:96]]
        l1, g1 = pm.grad(m, batch, "all")
        l2, g2 = pd.grad_dp(m, batch, "all")
        a, b = pm.flat_grads(g2).double(), pm.flat_grads(g1).double()
        out["grad_dp"] = bool((a - b).norm() <= 1e-6 * b.norm() and abs(float(l2) - l1) <= 1e-6 * l1
                              and l2.is_cuda) or f"grad rel {float((a - b).norm() / b.norm()):.2e} loss {float(l2)} {l1}"
    except Exception as e:  # report, do not hang the peer
        out["error"] = repr(e)
        raise
    finally:
        results[rank] = out
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_match_one_rank(cuda_device):
    port = _free_port()
    with mp.Manager() as manager:
        results = manager.dict()
        mp.spawn(_worker, args=(2, port, results), nprocs=2, join=True)
        res = dict(results)
    keys = ("sweep", "trainer_fo", "trainer_fo_stats", "trainer_so", "trainer_so_stats", "meta_step_dp",
            "meta_step_dp_stats", "grad_dp")
    for r in (0, 1):
        bad = {k: res[r].get(k) for k in keys if not res[r].get(k)}
        assert all(v is True for v in (res[r].get(k) for k in keys)), f"rank {r}: {res[r]}"
