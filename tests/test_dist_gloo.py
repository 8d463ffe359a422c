"""Multi-process (world_size 2, gloo, CPU) coverage of the data-parallel layer.

The device kernels are replaced by the oracle (tests may use it) through the
injectable compute callables; what is under test is the sharding, the
collectives and the merge semantics of dist.py.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import kt_oracle as ko
from paper_2102_04199_b200 import dist as pd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_merge(scores, idx, k):
    top = ko.rank_history(idx.numpy(), scores.numpy(), set(), k)
    sc = {int(i): float(s) for i, s in zip(idx.numpy(), scores.numpy())}
    return torch.tensor(top), torch.tensor([sc[i] for i in top], dtype=torch.float32)


def _scores_for(lo, count):
    # deterministic tie-heavy scores of config index i
    i = np.arange(lo, lo + count)
    return torch.tensor(np.round(np.sin(i * 0.37) * 4) / 4, dtype=torch.float32), torch.tensor(i)


def _worker(rank, world_size, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    try:
        # 1) sharded sweep + all-gathered top-k == single-process rank_history
        def score_topk(lo, count):
            s, i = _scores_for(lo, count)
            return _oracle_merge(s, i, 16)

        ti, ts = pd.sharded_sweep(score_topk, 1001, 16, base=5000, merge=_oracle_merge)
        s, i = _scores_for(5000, 1001)
        want = ko.rank_history(i.numpy(), s.numpy(), set(), 16)
        sweep_ok = ti.tolist() == want

        # 2) MAML data parallel (dist.meta_step_dp on a CPU ModelState; oracle task sums)
        from paper_2102_04199_b200.meta import MetaConfig
        from paper_2102_04199_b200.model import head_to_vec, init_model
        from paper_2102_04199_b200.util import rng_from

        m = init_model(rng_from("dp-model"), gcn_dims=(4,), head_hidden=(5,), device="cpu")
        shapes = [tuple(w.shape) for w in m.head.weights]
        theta = head_to_vec(m.head).double().numpy()
        rng = np.random.default_rng(0)
        tasks = [(rng.normal(size=(3, 8)), rng.normal(size=3), rng.normal(size=(3, 8)), rng.normal(size=3))
                 for _ in range(5)]

        def task_sum(local):
            g = np.zeros_like(theta)
            st = np.zeros(2)
            for us, ys, uq, yq in local:
                ls, lq, gi, _ = ko.maml_outer_grad(theta, lambda t: ko.head_loss_grad(t, shapes, us, ys),
                                                   lambda t: ko.head_loss_grad(t, shapes, uq, yq), 0.01, 1, True)
                g += gi
                st += [ls, lq]
            return torch.tensor(g, dtype=torch.float32), torch.tensor(st)

        cfg = MetaConfig(alpha=0.01, beta=0.001)
        m2, stats = pd.meta_step_dp(m, tasks, cfg, task_sum=task_sum)
        ref_theta, ref_ls, ref_lq = ko.meta_step_embedded(theta, shapes, tasks, 0.01, 0.001)
        maml_ok = np.allclose(head_to_vec(m2.head).double().numpy(), ref_theta, rtol=1e-6, atol=1e-7) and \
            np.allclose([stats["support_loss"], stats["query_loss"]], [ref_ls, ref_lq]) and \
            torch.equal(m2._flat[: 12 * 4 + 4], m._flat[: 12 * 4 + 4])

        # 3) grad data parallel: batch-mean over the union of shards
        batch = list(range(7))

        def local_grad(shard):
            v = torch.tensor([float(x) for x in shard], dtype=torch.float64)
            return float((v ** 2).mean()), torch.stack([v.mean(), (2 * v).mean()])

        loss, g = pd.grad_dp(object(), batch, local_grad=local_grad)
        full = torch.tensor(batch, dtype=torch.float64)
        grad_ok = abs(loss - float((full ** 2).mean())) < 1e-12 and \
            torch.allclose(g, torch.stack([full.mean(), (2 * full).mean()]))
        results[rank] = (sweep_ok, maml_ok, grad_ok)
    finally:
        dist.destroy_process_group()


def test_shard_bounds_cover_and_balance():
    for n in (0, 1, 7, 1000, 1 << 20):
        for ws in (1, 2, 3, 8):
            spans = [pd.shard_bounds(n, r, ws) for r in range(ws)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1


def test_world_size_two_gloo():
    port = _free_port()
    with mp.Manager() as manager:
        results = manager.dict()
        mp.spawn(_worker, args=(2, port, results), nprocs=2, join=True)
        assert dict(results) == {0: (True, True, True), 1: (True, True, True)}
