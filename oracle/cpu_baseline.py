"""TEST INFRASTRUCTURE: the timed CPU baseline (bench.py cpu_baseline / --impl reference).

Runs the oracle port of the reference's candidate-scoring path -- the
`meta_scores` closure (search.py:534-541): encode_batch (graphs.py:305) ->
embed_batch (model.py:185) -> head_forward_batch (model.py:197), fp64 numpy,
in 4,096-candidate chunks (the reference's C1 shape) -- on the host cores,
one process per core with single-threaded BLAS, candidates sharded by
contiguous chunk.  Never used by the product path.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import kt_oracle as ko

_STATE = {}


def _init(params, op, spec_args, super_graph):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    ext = ko.extents(op, *spec_args)
    knobs = ko.knob_lists(op, ext)
    adj, rows, mask = ko.layout(op, super_graph)
    _STATE.update(params=params, op=op, ext=ext, knobs=knobs, adj=adj, rows=rows, mask=mask,
                  cards=[len(v) for _, v in knobs])


def _score_chunk(idx):
    s = _STATE
    ch = ko.decode(s["cards"], idx)
    x = ko.encode(s["op"], s["ext"], s["knobs"], ch, s["adj"].shape[0], s["rows"])
    return ko.score(s["params"], x, s["mask"], s["adj"])


def score_indices(params, op, spec_args, super_graph, idx, chunk=4096):
    """Single-process oracle scores (fp64) for config indices."""
    _init(params, op, spec_args, super_graph)
    return np.concatenate([_score_chunk(idx[i : i + chunk]) for i in range(0, len(idx), chunk)])


class SweepPool:
    """Process pool (one process per usable core, single-threaded BLAS) scoring
    candidate chunks with the oracle; reused across timed steps."""

    def __init__(self, params, op, spec_args, super_graph, procs=None, chunk=4096):
        import multiprocessing as mp

        self.procs = procs or len(os.sched_getaffinity(0))
        self.chunk = chunk
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        self.pool = mp.get_context("spawn").Pool(self.procs, initializer=_init,
                                                 initargs=(params, op, spec_args, super_graph))
        rng = np.random.default_rng(0)
        self.pool.map(_score_chunk, [rng.integers(0, 1000, chunk) for _ in range(self.procs)])  # warm workers

    def time(self, idx):
        """(seconds, scores) for scoring idx across the pool."""
        chunks = [idx[i : i + self.chunk] for i in range(0, len(idx), self.chunk)]
        t0 = time.perf_counter()
        out = self.pool.map(_score_chunk, chunks, chunksize=max(1, len(chunks) // (4 * self.procs)))
        return time.perf_counter() - t0, np.concatenate(out)

    def close(self):
        self.pool.close()
        self.pool.join()


def time_sweep(params, op, spec_args, super_graph, idx, chunk=4096, procs=None, reps=1):
    """Best-of-reps wall time (s) of scoring `idx` on `procs` processes (default: all usable cores)."""
    sp = SweepPool(params, op, spec_args, super_graph, procs, chunk)
    try:
        best, out = float("inf"), None
        for _ in range(reps):
            secs, out = sp.time(idx)
            best = min(best, secs)
        return best, sp.procs, out
    finally:
        sp.close()


# --- secondary configs: C2 pretrain step, C3 meta_step, C4 fine-tune ---------------------
#
# BASELINE.md 2 / SURVEY.md 8(d): each GPU number sits beside the reference path timed on
# the box's host cores, (i) one process and (ii) P processes (P = usable cores) sharding the
# batch (C2) or the tasks (C3), single-threaded BLAS per process, min and median over >= 9
# repetitions.  The per-step work is the reference's own: C2 = grad (model.py:218, a
# per-graph fwd/bwd loop) + sgd_step (model.py:288); C3 = meta_step (meta.py:223-257), which
# re-embeds every support / query graph through the frozen GCN one graph at a time
# (`_embedded`, meta.py:199-208) before the head-only MAML math; C4 = fine_tune_embedded
# (meta.py:274-282) on the 64 x 64 embeddings (64 rows do not shard: 1 process only).


def graph_triple(op, spec_args, index, super_graph=True):
    """(X raw fp64, Â, mask) of one schedule graph, from the oracle encoder."""
    ext = ko.extents(op, *spec_args)
    knobs = ko.knob_lists(op, ext)
    adj, rows, mask = ko.layout(op, super_graph)
    ch = ko.decode([len(v) for _, v in knobs], np.array([index]))
    return ko.encode(op, ext, knobs, ch, adj.shape[0], rows)[0], adj, mask


_WORK = {}


def _work_init(kind, params, data):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    _WORK.update(kind=kind, params=params, data=data)


def _c2_shard(bounds):
    """Mean loss / grads of model.grad over graphs[lo:hi] (the shard's share of the batch)."""
    lo, hi = bounds
    graphs, labels = _WORK["data"]
    loss, g = ko.grad(_WORK["params"], graphs[lo:hi], labels[lo:hi])
    return hi - lo, loss, g


def _c3_shard(bounds):
    """Sum over tasks[lo:hi] of maml_outer_grad's g_i, with the reference's per-graph
    re-embedding of the support and query sets (meta.py:199-208, 223-257)."""
    lo, hi = bounds
    p = _WORK["params"]
    tasks, shapes, alpha, fo, theta = _WORK["data"]
    out, sl, ql = np.zeros_like(theta), 0.0, 0.0
    for sup, ys, qry, yq in tasks[lo:hi]:
        us = np.stack([ko.embed_batch(p, x[None], m, a)[0] for x, a, m in sup])
        uq = np.stack([ko.embed_batch(p, x[None], m, a)[0] for x, a, m in qry])
        ls, lq, g, _ = ko.maml_outer_grad(
            theta, lambda t: ko.head_loss_grad(t, shapes, us, ys), lambda t: ko.head_loss_grad(t, shapes, uq, yq),
            alpha, 1, fo, lambda t, v: ko.head_hvp(t, shapes, us, ys, v))
        out += g
        sl += ls
        ql += lq
    return out, sl, ql


def _combine_c2(parts, n):
    loss = sum(k * l for k, l, _ in parts) / n
    g = None
    for k, _, gs in parts:
        w = k / n
        if g is None:
            g = {key: ([a * w for a in v] if isinstance(v, list) else v * w) for key, v in gs.items()}
        else:
            for key, v in gs.items():
                if isinstance(v, list):
                    g[key] = [a + b * w for a, b in zip(g[key], v)]
                else:
                    g[key] = g[key] + v * w
    return loss, g


def _bounds(n, parts):
    step = -(-n // parts)
    return [(lo, min(n, lo + step)) for lo in range(0, n, step)]


def _stats(times):
    t = np.array(times) * 1e3
    return {"min_ms": float(t.min()), "median_ms": float(np.median(t)), "reps": len(times)}


def time_secondary(kind, params, data, reps=9, procs=None, lr=0.005, beta=0.001):
    """{"1proc": {min_ms, median_ms, reps}, "Pproc": {..., "procs": P}} for one step of
    C2 (kind "c2": data = (graphs, labels)) or C3 (kind "c3": data = (tasks, shapes,
    alpha, first_order, theta)); the update (sgd / theta - beta * sum) is in the step."""
    import multiprocessing as mp

    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    shard = _c2_shard if kind == "c2" else _c3_shard
    n = len(data[0])

    def finish(parts):
        if kind == "c2":
            _, g = _combine_c2(parts, n)
            return ko.sgd(params, g, lr)
        theta = data[4]
        return theta - beta * sum(p[0] for p in parts)

    out = {}
    _work_init(kind, params, data)
    times = []
    for _ in range(reps + 1):
        t0 = time.perf_counter()
        finish([shard((0, n))])
        times.append(time.perf_counter() - t0)
    out["1proc"] = _stats(times[1:])
    procs = procs or len(os.sched_getaffinity(0))
    procs = min(procs, n)
    pool = mp.get_context("spawn").Pool(procs, initializer=_work_init, initargs=(kind, params, data))
    try:
        b = _bounds(n, procs)
        times = []
        for _ in range(reps + 1):
            t0 = time.perf_counter()
            finish(pool.map(shard, b, chunksize=1))
            times.append(time.perf_counter() - t0)
        out["Pproc"] = dict(_stats(times[1:]), procs=len(b))
    finally:
        pool.close()
        pool.join()
    return out


def time_fine_tune(theta, shapes, u, y, alpha=0.01, steps=8, reps=9):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    times = []
    for _ in range(reps + 1):
        t0 = time.perf_counter()
        ko.fine_tune_embedded(theta, shapes, u, y, alpha, steps)
        times.append(time.perf_counter() - t0)
    return {"1proc": _stats(times[1:])}


def host_info() -> dict:
    """CPU model, usable cores, numpy / BLAS versions of the timing host."""
    import platform
    import subprocess

    info = {"cores": len(os.sched_getaffinity(0)), "numpy": np.__version__, "python": platform.python_version()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
            elif line.startswith("CPU(s):"):
                info["cpus"] = int(line.split(":", 1)[1])
    except (OSError, ValueError, subprocess.SubprocessError):
        pass
    try:
        cfg = np.show_config(mode="dicts")
        blas = cfg["Build Dependencies"]["blas"]
        info["blas"] = f"{blas.get('name')} {blas.get('version')}"
    except Exception:  # noqa: BLE001 -- informational only
        pass
    return info
