"""Data parallelism for the cost-model path (one process per GPU, torch.distributed).

The reference is single-process; its parallel axes are the
candidate set and the MAML task batch:
  * candidate scoring shards contiguous index ranges over ranks with no
    collective on the data path; the only exchange is the ranking: each rank's
    top-k (k x {fp32 score, int64 index}) is all-gathered and merged by
    (score desc, index asc) -- identical to rank_history over the union because
    the scorer is position-invariant;
  * a MAML outer step shards the task list; every rank computes the outer gradients
    g_i of its contiguous task share (kt_maml_task_grads), the per-task rows are
    all-gathered in task order (T x 8,385 fp32, 1 MB at 32 tasks) and every rank sums
    all of them in task order and applies theta - beta * sum ("sum, not mean",
    meta.py:226-252) -- bit-identical to the one-GPU kt_maml_step for any world size;
  * a pretrain / grad step shards the batch; per-rank gradient sums scaled by
    b_local / B are all-reduced so the result is the full-batch mean.
NCCL over NVLink carries these on B200 nodes (and can be captured in a CUDA graph);
on gloo -- the CPU test backend, also used to run several ranks on one GPU -- device
tensors are staged through host memory.  Compute callables are injectable so the host
logic is testable without a GPU.
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


def _staged(t: torch.Tensor, group=None) -> bool:
    """Device tensor on a backend without device collectives (gloo): go through the host."""
    return t.is_cuda and dist.get_backend(group) != "nccl"


def all_gather_rows(out: torch.Tensor, inp: torch.Tensor, group=None) -> torch.Tensor:
    """out (world * n, ...) <- every rank's inp (n, ...), in rank order."""
    _, ws = world()
    if ws == 1:
        return out.copy_(inp)
    if not _staged(inp, group) and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp.contiguous(), group=group)
        return out
    parts = [torch.empty(inp.shape, dtype=inp.dtype) for _ in range(ws)]
    dist.all_gather(parts, inp.detach().cpu().contiguous(), group=group)
    return out.copy_(torch.cat(parts).reshape(out.shape))


def allgather_topk(top_idx: torch.Tensor, top_score: torch.Tensor, k: int, merge=None, group=None):
    """Global top-k from per-rank top-k lists: all-gather, then merge by (score desc, index asc).

    `merge(scores, indices, k) -> (idx, scores)`; defaults to the device kernel
    search.topk_merge."""
    _, ws = world()
    if ws == 1:
        return top_idx, top_score
    gs = torch.empty(ws * top_score.numel(), dtype=top_score.dtype, device=top_score.device)
    gi = torch.empty(ws * top_idx.numel(), dtype=top_idx.dtype, device=top_idx.device)
    all_gather_rows(gs, top_score, group)
    all_gather_rows(gi, top_idx, group)
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
        if _staged(t, group):
            h = t.detach().cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def meta_step_dp(m, tasks: list, cfg, *, task_sum=None, group=None):
    """Data-parallel meta_step: this rank's contiguous task share; bit-identical to meta_step.

    Every rank must pass the identical task list (sampled from identically seeded host
    RNGs); all ranks return the same model.  Device path: per-task gradient rows
    (kt_maml_task_grads), all-gathered in task order (shares padded with zero rows to
    equal length: adding +0.0 leaves an fp64 sum unchanged), then the fixed-order fp64
    task sum and the outer update (kt_task_sum_update) -- the arithmetic of kt_maml_step.
    `task_sum(local) -> (g_sum, (sum ls, sum lq))` replaces the device path (CPU tests)."""
    from .meta import _embedded, _task_index
    from .model import dims_of, head_to_vec, with_head_vec

    if not tasks:
        raise DomainError("empty task batch")
    rank, ws = world()
    local = shard_list(tasks, rank, ws)
    theta = head_to_vec(m.head)
    if task_sum is not None:  # injected host compute: all-reduce of the per-rank sums
        g_sum, stats = task_sum(local)
        allreduce_sum_(g_sum, group)
        allreduce_sum_(stats, group)
        st = stats.cpu().numpy() / len(tasks)
        new = theta - cfg.beta * g_sum
        return with_head_vec(m, new), {"support_loss": float(st[0]), "query_loss": float(st[1])}
    from . import _lib

    d = dims_of(m)
    dev = theta.device
    P = d.n_head_params
    per = -(-len(tasks) // ws)  # equal shares for the all-gather
    rows = torch.zeros((per, P), dtype=torch.float32, device=dev)
    losses = torch.zeros((per, 2), dtype=torch.float32, device=dev)
    lib = _lib.load()
    if local:
        uniq, s_off, s_idx, q_off, q_idx = _task_index(local)
        u, y = _embedded(m, uniq)
        # (the index tensors must outlive the launch: keep references, not bare pointers)
        so, si, qo, qi = (torch.tensor(a, dtype=torch.int64, device=dev) for a in (s_off, s_idx, q_off, q_idx))
        T = len(local)
        ws_bytes = int(lib.kt_maml_workspace_bytes(d, T, cfg.inner_steps, int(cfg.first_order)))
        wsp = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        with torch.cuda.device(dev):
            _lib.check(lib.kt_maml_task_grads(d, _lib.ptr(theta), _lib.ptr(u), _lib.ptr(y), _lib.ptr(so),
                                              _lib.ptr(si), _lib.ptr(qo), _lib.ptr(qi), T,
                                              float(cfg.alpha), int(cfg.inner_steps), int(cfg.first_order),
                                              _lib.ptr(rows), _lib.ptr(losses), _lib.ptr(wsp), ws_bytes,
                                              _lib.stream_handle()), "meta task grads")
    all_rows = torch.empty((per * ws, P), dtype=torch.float32, device=dev)
    all_losses = torch.empty((per * ws, 2), dtype=torch.float32, device=dev)
    all_gather_rows(all_rows, rows, group)
    all_gather_rows(all_losses, losses, group)
    new = theta.clone()
    g_sum = torch.empty(P, dtype=torch.float32, device=dev)
    stats = torch.empty(2, dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        _lib.check(lib.kt_task_sum_update(d, _lib.ptr(all_rows), _lib.ptr(all_losses), per * ws, float(cfg.beta),
                                          _lib.ptr(new), _lib.ptr(g_sum), _lib.ptr(stats), _lib.stream_handle()),
                   "meta outer update")
    st = stats.cpu().numpy() / len(tasks)
    return with_head_vec(m, new), {"support_loss": float(st[0]), "query_loss": float(st[1])}


def grad_dp(m, batch: list, scope: str = "all", *, local_grad=None, group=None):
    """Data-parallel grad: batch mean over the union of the ranks' shards.

    Device-resident: returns (loss, grads) with the loss a 0-d fp64 tensor on the
    gradients' device (no host synchronisation; `float(loss)` when needed).
    `local_grad(shard) -> (loss_mean tensor, flat_grad_mean)` (the device grad kernel on
    the shard in production)."""
    from .model import _grad_packed, grads_from_flat, normalize_label, pack_graphs, flat_params

    if not batch:
        raise DomainError("empty batch")
    rank, ws = world()
    local = shard_list(batch, rank, ws)
    frac = len(local) / len(batch)
    if local_grad is None:
        def local_grad(shard):
            import numpy as np

            ys = np.array([normalize_label(m, float(v)) for _, v in shard], dtype=np.float32)
            dev = flat_params(m).device
            pk = pack_graphs([g for g, _ in shard], dev)
            loss, g, _ = _grad_packed(m, pk, torch.from_numpy(ys).to(dev), scope)
            return loss.reshape(()), g
    if local:
        loss, g = local_grad(local)
        g = g * frac
        lt = torch.as_tensor(loss, dtype=torch.float64, device=g.device).reshape(1) * frac
    else:
        g0 = local_grad(batch[:1])[1]
        g = torch.zeros_like(g0)
        lt = torch.zeros(1, dtype=torch.float64, device=g.device)
    allreduce_sum_(g, group)
    allreduce_sum_(lt, group)
    return lt.reshape(()), (grads_from_flat(g, m) if hasattr(m, "gcn") else g)
