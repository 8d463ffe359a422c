"""Data parallelism for the cost-model path (one process per GPU, torch.distributed).

The reference is single-process; its parallel axes are the
candidate set and the MAML task batch:
  * candidate scoring shards contiguous index ranges over ranks with no
    collective on the data path; the only exchange is the ranking: each rank's
    top-k (k x {fp32 score, int64 index}) is all-gathered and merged by
    (score desc, index asc) -- identical to rank_history over the union because
    the scorer is position-invariant;
  * a MAML outer step shards the task list; the per-rank sums of g_i are
    all-reduced (SUM) and every rank applies the same theta - beta * sum
    ("sum, not mean", meta.py:226-252);
  * a pretrain / grad step shards the batch; per-rank gradient sums scaled by
    b_local / B are all-reduced so the result is the full-batch mean.
NCCL over NVLink carries these on B200 nodes; the same code runs on gloo (CPU)
in the tests.  Compute callables are injectable so the host logic is testable
without a GPU.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .errors import DomainError


def world() -> tuple:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_bounds(n: int, rank: int, world_size: int) -> tuple:
    """Contiguous [lo, hi) share of n items for `rank` (sizes differ by at most one)."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise DomainError("bad rank / world size")
    base, extra = divmod(n, world_size)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_list(items: list, rank: int, world_size: int) -> list:
    lo, hi = shard_bounds(len(items), rank, world_size)
    return items[lo:hi]


def allgather_topk(top_idx: torch.Tensor, top_score: torch.Tensor, k: int, merge=None, group=None):
    """Global top-k from per-rank top-k lists: all-gather, then merge by (score desc, index asc).

    `merge(scores, indices, k) -> (idx, scores)`; defaults to the device kernel
    search.topk_merge."""
    _, ws = world()
    if ws == 1:
        return top_idx, top_score
    gs = torch.empty(ws * top_score.numel(), dtype=top_score.dtype, device=top_score.device)
    gi = torch.empty(ws * top_idx.numel(), dtype=top_idx.dtype, device=top_idx.device)
    dist.all_gather_into_tensor(gs, top_score.contiguous(), group=group)
    dist.all_gather_into_tensor(gi, top_idx.contiguous(), group=group)
    if merge is None:
        from .search import topk_merge as merge
    return merge(gs, gi, k)


def sharded_sweep(score_topk, n_total: int, k: int, *, base: int = 0, merge=None, group=None):
    """Score candidates [base, base + n_total) sharded over ranks and return the global top-k.

    `score_topk(lo, count) -> (top_idx, top_score)` scores a contiguous shard on
    this rank (Sweeper.run_device in production)."""
    rank, ws = world()
    lo, hi = shard_bounds(n_total, rank, ws)
    ti, ts = score_topk(base + lo, hi - lo)
    return allgather_topk(ti, ts, k, merge=merge, group=group)


def allreduce_sum_(t: torch.Tensor, group=None) -> torch.Tensor:
    _, ws = world()
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def meta_step_dp(m, tasks: list, cfg, *, task_sum=None, group=None):
    """Data-parallel meta_step: this rank's contiguous task shard, all-reduced sum.

    Every rank must pass the identical task list (sampled from identically seeded
    host RNGs); all ranks return the same model."""
    from .meta import _embedded, _sgd, _task_index, maml_sum
    from .model import head_to_vec, with_head_vec

    if not tasks:
        raise DomainError("empty task batch")
    rank, ws = world()
    local = shard_list(tasks, rank, ws)
    theta = head_to_vec(m.head)
    if task_sum is not None:
        g_sum, stats = task_sum(local)
    elif local:
        uniq, s_off, s_idx, q_off, q_idx = _task_index(local)
        u, y = _embedded(m, uniq)
        up = lambda a: torch.tensor(a, dtype=torch.int64, device=u.device)
        g_sum, stats = maml_sum(m, u, y, up(s_off), up(s_idx), up(q_off), up(q_idx), cfg)
    else:
        g_sum = torch.zeros_like(theta)
        stats = torch.zeros(2, dtype=torch.float64, device=theta.device)
    allreduce_sum_(g_sum, group)
    allreduce_sum_(stats, group)
    st = stats.cpu().numpy() / len(tasks)
    new = _sgd(theta, g_sum, cfg.beta) if theta.is_cuda else theta - cfg.beta * g_sum
    return with_head_vec(m, new), {"support_loss": float(st[0]), "query_loss": float(st[1])}


def grad_dp(m, batch: list, scope: str = "all", *, local_grad=None, group=None):
    """Data-parallel grad: batch mean over the union of the ranks' shards.

    `local_grad(shard) -> (loss_mean, flat_grad_mean)` (model.grad in production)."""
    from .model import flat_grads, grad, grads_from_flat

    if not batch:
        raise DomainError("empty batch")
    rank, ws = world()
    local = shard_list(batch, rank, ws)
    frac = len(local) / len(batch)
    if local_grad is None:
        def local_grad(shard):
            loss, g = grad(m, shard, scope)
            return loss, flat_grads(g)
    if local:
        loss, g = local_grad(local)
        g = g * frac
        lt = torch.tensor([loss * frac], dtype=torch.float64, device=g.device)
    else:
        g0 = local_grad(batch[:1])[1]
        g = torch.zeros_like(g0)
        lt = torch.zeros(1, dtype=torch.float64, device=g.device)
    allreduce_sum_(g, group)
    allreduce_sum_(lt, group)
    return float(lt.item()), (grads_from_flat(g, m) if hasattr(m, "gcn") else g)
