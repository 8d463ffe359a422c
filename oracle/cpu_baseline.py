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
