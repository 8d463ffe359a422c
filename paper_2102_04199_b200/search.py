"""The predictor seam of the tuner, on the GPU.

The reference's proposers take the cost model as a plain callable
`predict(list[KnobConfig]) -> scores` (search.py:9-10, sa_explore 202-254), and
`tune` builds it as meta_scores / meta_energy = encode_batch -> embed_batch ->
head_forward_batch (search.py:534-541).  `CostModelPredictor` is that callable
backed by the fused sm_100a scorer (kt_score_indices), and `rank_history`
keeps the reference's (-score, index) ordering (search.py:257-264).  For large
candidate sets `score_indices` + `topk` stay on the device end to end.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import DomainError, NumericError
from .graphs import BatchLayout, batch_layout, configs_to_indices, device_spec_table
from .kernels import KernelSpec, KnobSpace
from .model import ModelState, dims_of, flat_params

DEFAULT_DIMS = (12, (32, 32), (64, 64))


def _default_model(m: ModelState) -> bool:
    d = dims_of(m)
    return (d.F, tuple(d.gcn[1 : d.n_gcn + 1]), tuple(d.head[1 : d.n_head])) == DEFAULT_DIMS


def score_indices(m: ModelState, spec: KernelSpec, space: KnobSpace, layout: BatchLayout, idx=None, *,
                  base: int = 0, count: int | None = None, want_u: bool = False, check: bool = True,
                  z_out=None, u_out=None, err=None, engine: str = "tc"):
    """Scores z (fp32 device, normalised log2 GFLOPS) of config indices.

    `idx` is an int64 device tensor (or array-like); with idx=None the candidates
    are the contiguous range [base, base+count).  Equals
    head_forward_batch(embed_batch(m, encode_batch(...), mask, adj), head).
    engine "tc": tcgen05 3xTF32 kernel (kt_score_indices); "fp32": FFMA2 kernel.
    """
    flat = flat_params(m)
    dev = flat.device
    if not _default_model(m) or space.size >= 2**32:
        return _score_general(m, spec, space, layout, idx, base, count, want_u)
    if idx is not None and not isinstance(idx, torch.Tensor):
        idx = torch.from_numpy(np.ascontiguousarray(idx, dtype=np.int64)).to(dev)
    b = int(idx.numel()) if idx is not None else int(count or 0)
    if b <= 0:
        raise DomainError("empty batch")
    tab = device_spec_table(spec, space, layout, m.feature_norm.mean, m.feature_norm.std, device=dev)
    z = z_out if z_out is not None else torch.empty(b, dtype=torch.float32, device=dev)
    u = None
    if want_u:
        u = u_out if u_out is not None else torch.empty((b, 64), dtype=torch.float32, device=dev)
    e = err if err is not None else torch.zeros(1, dtype=torch.int32, device=dev)
    lib = _lib.load()
    with torch.cuda.device(dev):
        fn = lib.kt_score_indices if engine == "tc" else lib.kt_score_indices_fp32
        _lib.check(fn(_lib.ptr(tab), dims_of(m), _lib.ptr(flat), _lib.ptr(idx), base, b, _lib.ptr(z), _lib.ptr(u),
                      _lib.ptr(e), _lib.stream_handle()), "score_indices")
    if check and int(e.item()):
        raise DomainError("config index out of range for the knob space")
    return (z, u) if want_u else z


def _score_general(m, spec, space, layout, idx, base, count, want_u):
    from .graphs import encode_batch
    from .model import embed_batch, head_forward_batch

    dev = flat_params(m).device
    if idx is None:
        idx = torch.arange(base, base + int(count), dtype=torch.int64, device=dev)
    feats = encode_batch(spec, space, idx, layout, device=dev)
    u = embed_batch(m, feats, layout.feature_mask, layout.adjacency)
    z = head_forward_batch(u, m.head)
    return (z, u) if want_u else z


class CostModelPredictor:
    """`predict(configs) -> np.ndarray` for sa_explore / tune (search.py:202-254, 534-541).

    `meta_scores(configs)` returns (z, u) like the reference closure; both are
    host numpy arrays (float64 scores in input order), so this object is a
    drop-in wherever the reference passes `meta_energy`.
    """

    def __init__(self, m: ModelState, spec: KernelSpec, space: KnobSpace, layout: BatchLayout | None = None,
                 template=None):
        self.m = m
        self.spec = spec
        self.space = space
        self.layout = layout if layout is not None else batch_layout(spec, template)

    def _fast(self, idx: np.ndarray, want_u: bool):
        """Pre-resolved launch for the default dims (spec table, dims and parameter pointer
        looked up once per model object; pinned staging for the indices and scores)."""
        m = self.m
        st = getattr(self, "_st", None)
        if st is None or st["m"] is not m:
            flat = flat_params(m)
            st = self._st = {"m": m, "flat": flat, "dims": dims_of(m), "dev": flat.device,
                             "tab": device_spec_table(self.spec, self.space, self.layout, m.feature_norm.mean,
                                                      m.feature_norm.std, device=flat.device),
                             "err": torch.zeros(1, dtype=torch.int32, device=flat.device), "cap": 0}
        b = idx.size
        if st["cap"] < b:
            cap = max(b, 2 * st["cap"])
            st["h_idx"] = torch.empty(cap, dtype=torch.int64, pin_memory=True)
            st["h_idx32"] = torch.empty(cap, dtype=torch.int32, pin_memory=True)
            st["d_idx"] = torch.empty(cap, dtype=torch.int64, device=st["dev"])
            st["z"] = torch.empty(cap, dtype=torch.float32, device=st["dev"])
            st["h_z"] = torch.empty(cap, dtype=torch.float32, pin_memory=True)
            st["cap"] = cap
        lib = _lib.load()
        if not want_u:
            # scores only: the scorer reads the uint32 indices from pinned host memory and writes
            # the scores back into pinned host memory in place (zero-copy, no copy launches)
            st["h_idx32"][:b].numpy().view(np.uint32)[:] = idx
            with torch.cuda.device(st["dev"]):
                _lib.check(lib.kt_score_indices_ex(_lib.ptr(st["tab"]), st["dims"], _lib.ptr(st["flat"]), None,
                                                   st["h_idx32"].data_ptr(), 0, b, st["h_z"].data_ptr(), None, None,
                                                   None, _lib.ptr(st["err"]), _lib.stream_handle()), "predict")
                torch.cuda.current_stream().synchronize()
            return st["h_z"][:b].numpy().astype(np.float64), None
        st["h_idx"][:b].numpy()[:] = idx
        u = torch.empty((b, 64), dtype=torch.float32, device=st["dev"])
        with torch.cuda.device(st["dev"]):
            st["d_idx"][:b].copy_(st["h_idx"][:b], non_blocking=True)
            _lib.check(lib.kt_score_indices(_lib.ptr(st["tab"]), st["dims"], _lib.ptr(st["flat"]),
                                            _lib.ptr(st["d_idx"]), 0, b, _lib.ptr(st["z"]), _lib.ptr(u),
                                            _lib.ptr(st["err"]), _lib.stream_handle()), "predict")
            st["h_z"][:b].copy_(st["z"][:b], non_blocking=True)
            torch.cuda.current_stream().synchronize()
        return st["h_z"][:b].numpy().astype(np.float64), u

    def meta_scores(self, configs):
        idx = configs_to_indices(self.space, configs)
        if _default_model(self.m) and self.space.size < 2**32 and idx.size:
            z, u = self._fast(idx, True)
            return z, u.double().cpu().numpy()
        z, u = score_indices(self.m, self.spec, self.space, self.layout, idx, want_u=True, check=False)
        return z.double().cpu().numpy(), u.double().cpu().numpy()

    def __call__(self, configs) -> np.ndarray:
        idx = configs_to_indices(self.space, configs)
        if _default_model(self.m) and self.space.size < 2**32 and idx.size:
            return self._fast(idx, False)[0]
        z = score_indices(self.m, self.spec, self.space, self.layout, idx, check=False)
        return z.double().cpu().numpy()


def rank_history(history: dict, visited: set, count: int) -> list:
    """Best `count` unvisited indices, highest score first, ties -> lower index."""
    ranked = sorted(((i, e) for i, e in history.items() if i not in visited), key=lambda t: (-t[1], t[0]))
    return [i for i, _ in ranked[:count]]


def topk(scores: torch.Tensor, k: int, idx: torch.Tensor | None = None, *, base: int = 0, visited=None):
    """Device rank_history: the k best (score desc, index asc) candidates, visited excluded.

    Returns (indices int64, scores fp32) device tensors of length k (index -1 pads
    when fewer than k candidates survive)."""
    dev = scores.device
    b = scores.numel()
    if b == 0:
        raise DomainError("empty candidate set")
    # the device keys pack the candidate index into 32 bits (score desc, index asc)
    if idx is None:
        if base < 0 or base + b > 2**32:
            raise DomainError("topk ranks candidate indices below 2^32")
    elif idx.dtype == torch.int64 and b and (int(idx.max()) >= 2**32 or int(idx.min()) < 0):
        raise DomainError("topk ranks candidate indices below 2^32")
    vis = None
    if visited:
        vis = torch.from_numpy(np.array(sorted(int(v) for v in visited), dtype=np.int64)).to(dev)
    lib = _lib.load()
    ws_bytes = int(lib.kt_topk_workspace_bytes(b, k))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    ti = torch.empty(k, dtype=torch.int64, device=dev)
    ts = torch.empty(k, dtype=torch.float32, device=dev)
    with torch.cuda.device(dev):
        _lib.check(lib.kt_topk(_lib.ptr(scores), _lib.ptr(idx), base, b, _lib.ptr(vis),
                               0 if vis is None else vis.numel(), k, _lib.ptr(ti), _lib.ptr(ts), _lib.ptr(ws),
                               ws_bytes, _lib.stream_handle()), "topk")
    return ti, ts


def topk_merge(scores: torch.Tensor, idx: torch.Tensor, k: int):
    """Merge concatenated per-rank (score, index) top-k lists into the global top-k."""
    dev = scores.device
    n = scores.numel()
    lib = _lib.load()
    ws_bytes = int(lib.kt_topk_workspace_bytes(n, k))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    ti = torch.empty(k, dtype=torch.int64, device=dev)
    ts = torch.empty(k, dtype=torch.float32, device=dev)
    with torch.cuda.device(dev):
        _lib.check(lib.kt_topk_merge(_lib.ptr(scores), _lib.ptr(idx), n, k, _lib.ptr(ti), _lib.ptr(ts),
                                     _lib.ptr(ws), ws_bytes, _lib.stream_handle()), "topk_merge")
    return ti, ts


class Sweeper:
    """Candidate-scoring sweep (C5): score a shard of config indices and keep the
    top-k by (score desc, index asc) -- rank_history over the whole shard.

    Everything per call is pre-resolved (spec table, dims, flat params, device
    buffers, streams), so a step is one or two C-ABI calls.  The scorer writes the
    64-bit (score, index) keys the radix top-k ranks, so the top-k never re-reads
    scores or indices.  `run_device` takes device-resident indices; `run_host` is
    the end-to-end form: pinned host indices in (read in place by the scorer),
    host scores + top-k out.
    """

    def __init__(self, m: ModelState, spec: KernelSpec, space: KnobSpace, layout: BatchLayout,
                 max_batch: int, k: int = 512):
        if not _default_model(m) or space.size >= 2**32:
            raise DomainError("Sweeper needs the default model dims and a space < 2^32 (use score_indices)")
        self.lib = _lib.load()
        self.flat = flat_params(m)
        self.dev = self.flat.device
        self.dims = dims_of(m)
        self.tab = device_spec_table(spec, space, layout, m.feature_norm.mean, m.feature_norm.std,
                                     device=self.dev)
        self.space_size = space.size
        self.max_batch, self.k = max_batch, k
        dev = self.dev
        self.z = torch.empty(max_batch, dtype=torch.float32, device=dev)
        self.keys = torch.empty(max_batch, dtype=torch.int64, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ws_bytes = int(self.lib.kt_topk_workspace_bytes(max_batch, k))
        self.ws = torch.zeros(self.ws_bytes, dtype=torch.uint8, device=dev)  # (its histogram starts at zero)
        self.top_idx = torch.empty(k, dtype=torch.int64, device=dev)
        self.top_score = torch.empty(k, dtype=torch.float32, device=dev)
        # two host result slots, so one end-to-end step can be in flight while the caller
        # consumes the previous one (submit / wait)
        self.h_z = torch.empty((2, max_batch), dtype=torch.float32, pin_memory=True)
        self.h_top_idx = torch.empty((2, k), dtype=torch.int64, pin_memory=True)
        self.h_top_score = torch.empty((2, k), dtype=torch.float32, pin_memory=True)
        self.ev_slot = [torch.cuda.Event(), torch.cuda.Event()]
        self._next_slot = 0
        self._pending = [None, None]  # per slot: (ticket, n) of the step in flight
        self._tickets = 0
        self._p = dict(tab=self.tab.data_ptr(), flat=self.flat.data_ptr(), err=self.err.data_ptr(),
                       ws=self.ws.data_ptr(), ti=self.top_idx.data_ptr(), ts=self.top_score.data_ptr(),
                       z=self.z.data_ptr(), keys=self.keys.data_ptr(),
                       hist=self.lib.kt_topk_key_hist(self.ws.data_ptr()))

    def score(self, idx64_ptr, idx32_ptr, base: int, n: int, stream) -> None:
        """The scorer launch alone: z[:n] and keys[:n] (raw pointers; bench timing hook)."""
        p = self._p
        _lib.check(self.lib.kt_score_indices_ex(p["tab"], self.dims, p["flat"], idx64_ptr, idx32_ptr, base, n,
                                                p["z"], None, p["keys"], p["hist"], p["err"], stream), "sweep score")

    def rank(self, n: int, stream) -> None:
        """Top-k of keys[:n] into top_idx / top_score (the scorer filled the first digit's bins)."""
        p = self._p
        _lib.check(self.lib.kt_topk_keys(p["keys"], n, self.k, 1, p["ti"], p["ts"], p["ws"], self.ws_bytes, stream),
                   "sweep topk")

    def run_device(self, idx: torch.Tensor | None = None, *, base: int = 0, count: int | None = None,
                   visited: torch.Tensor | None = None):
        """Scores into self.z[:n]; returns (top_idx, top_score) device views.  `idx`:
        int64 or int32 device indices, or None for base + arange(count)."""
        n = idx.numel() if idx is not None else int(count)
        if n > self.max_batch or n <= 0:
            raise DomainError("sweep batch size out of range")
        if idx is not None and idx.dtype not in (torch.int64, torch.int32):
            raise DomainError("sweep indices must be int64 or int32")
        st = torch.cuda.current_stream(self.dev).cuda_stream
        i64 = idx.data_ptr() if idx is not None and idx.dtype == torch.int64 else None
        i32 = idx.data_ptr() if idx is not None and idx.dtype == torch.int32 else None
        p = self._p
        if visited is None:
            self.score(i64, i32, base, n, st)
            self.rank(n, st)
        else:  # exclusion list: the top-k rebuilds keys from scores and tests membership
            if i32 is not None:
                raise DomainError("visited exclusion takes int64 indices")
            _lib.check(self.lib.kt_score_indices(p["tab"], self.dims, p["flat"], i64, base, n, p["z"], None,
                                                 p["err"], st), "sweep score")
            _lib.check(self.lib.kt_topk(p["z"], i64, base, n, visited.data_ptr(), visited.numel(), self.k, p["ti"],
                                        p["ts"], p["ws"], self.ws_bytes, st), "sweep topk")
        return self.top_idx, self.top_score

    def submit(self, idx_host: torch.Tensor) -> int:
        """Enqueue one end-to-end step (pinned host indices -> host scores + top-k) and
        return at once with a ticket; `wait(ticket)` returns its results.  Two steps may
        be in flight (the host result buffers alternate).

        int64 or int32 indices (the spaces this path takes are below 2^32).  One native
        call (kt_sweep_host): the scorer reads the pinned indices and writes the pinned
        scores in place over PCIe (int32 halves the index bytes), then the top-k."""
        n = idx_host.numel()
        if n > self.max_batch or n <= 0:
            raise DomainError("sweep batch size out of range")
        if idx_host.dtype not in (torch.int64, torch.int32):
            raise DomainError("sweep indices must be int64 or int32")
        if not idx_host.is_pinned():
            raise DomainError("run_host needs pinned host indices (torch pin_memory)")
        slot = self._next_slot
        if self._pending[slot] is not None:
            raise DomainError("two sweep steps already in flight: wait() for the older one first")
        comp = torch.cuda.current_stream(self.dev)
        p = self._p
        _lib.check(self.lib.kt_sweep_host(p["tab"], self.dims, p["flat"], idx_host.data_ptr(),
                                          idx_host.element_size(), n, p["keys"], self.h_z[slot].data_ptr(),
                                          self.k, p["ti"], p["ts"], self.h_top_idx[slot].data_ptr(),
                                          self.h_top_score[slot].data_ptr(), p["ws"], self.ws_bytes, p["err"],
                                          comp.cuda_stream), "sweep (host)")
        self.ev_slot[slot].record(comp)
        self._tickets += 1
        self._pending[slot] = (self._tickets, n)
        self._next_slot ^= 1
        return self._tickets

    def wait(self, ticket: int, check: bool = True):
        """Results of a submitted step: (host scores, host top-k idx, top-k scores).  The
        views stay valid until the step submitted after the next one reuses the slot."""
        slot = next((i for i, p in enumerate(self._pending) if p is not None and p[0] == ticket), None)
        if slot is None:
            raise DomainError(f"no step in flight for ticket {ticket} (already consumed or never submitted)")
        n = self._pending[slot][1]
        self.ev_slot[slot].synchronize()
        self._pending[slot] = None
        if check and int(self.err.item()):
            raise DomainError("config index out of range for the knob space")
        return self.h_z[slot, :n], self.h_top_idx[slot], self.h_top_score[slot]

    def run_host(self, idx_host: torch.Tensor, check: bool = True):
        """End to end, synchronously: submit + wait."""
        return self.wait(self.submit(idx_host), check)


# --- simulated-annealing exploration (search.py:177-281), the tuner's caller of the model ------


@dataclass
class SaSchedule:
    """search.py:48-59, same defaults and validation."""
    initial_temp: float = 1.0
    cooling: float = 0.95
    steps_per_round: int = 128
    parallel_chains: int = 16

    def __post_init__(self):
        if not 0.0 < self.cooling < 1.0:
            raise DomainError("cooling must be in (0, 1)")
        if self.initial_temp <= 0:
            raise DomainError("initial_temp must be positive")


def _space_multipliers(space: KnobSpace) -> np.ndarray:
    cards = [len(k.values) for k in space.knobs]
    mult = np.ones(len(cards), dtype=np.int64)
    for j in range(len(cards) - 2, -1, -1):
        mult[j] = mult[j + 1] * cards[j + 1]
    return mult


def draw_unvisited(space: KnobSpace, visited: set, count: int, rng) -> list:
    """Distinct config indices outside `visited`, uniform (search.py:185-211): the same
    numpy Generator calls as the reference, so a shared seed gives the same indices."""
    size = space.size
    remaining = size - len(visited)
    count = min(count, max(remaining, 0))
    if count <= 0:
        return []
    if size <= 65536:
        unvisited = np.array([i for i in range(size) if i not in visited], dtype=np.int64)
        pick = rng.choice(len(unvisited), size=count, replace=False)
        return [int(unvisited[i]) for i in pick]
    out: list = []
    chosen: set = set()
    guard = 0
    while len(out) < count:
        need = count - len(out)
        for v in rng.integers(0, size, size=need + 8):
            i = int(v)
            if i not in visited and i not in chosen:
                chosen.add(i)
                out.append(i)
                if len(out) == count:
                    break
        guard += 1
        if guard > 10000:
            raise NumericError("unvisited sampling failed to converge")
    return out


class DeviceAnnealer:
    """sa_explore's chains on the GPU for one CostModelPredictor.

    The per-step random draws come from the caller's Generator in the reference's order
    (they never depend on the predictions: kt_sa_draws).  engine "fused" (default, up to
    128 chains): the whole annealing loop is one kt_sa_run launch -- the fused scorer on
    one CTA proposes, scores and accepts step after step.  engine "steps": every step is
    kt_sa_propose -> scorer -> kt_sa_accept on device-resident chain state, the step
    sequence captured once into a CUDA graph and replayed.  Both give the reference
    loop's history."""

    def __init__(self, predictor: CostModelPredictor, sched: SaSchedule, n_chains: int, engine: str | None = None):
        m, space = predictor.m, predictor.space
        if not _default_model(m) or space.size >= 2**32:
            raise DomainError("device annealing needs the default model dims and a space < 2^32")
        self.pred, self.sched, self.n = predictor, sched, n_chains
        self.m = m
        self.lib = _lib.load()
        self.flat = flat_params(m)
        dev = self.dev = self.flat.device
        self.dims = dims_of(m)
        self.tab = device_spec_table(predictor.spec, space, predictor.layout, m.feature_norm.mean,
                                     m.feature_norm.std, device=dev)
        self.cards_np = np.array([len(k.values) for k in space.knobs], dtype=np.int64)
        self.nk = len(self.cards_np)
        self.cards = torch.from_numpy(self.cards_np.astype(np.int32)).to(dev)
        self.mult = torch.from_numpy(_space_multipliers(space)).to(dev)
        steps, n, nk = sched.steps_per_round, n_chains, self.nk
        # the step draws (u, knob, delta, resample, nudge) as views of one byte buffer, host
        # (pinned) and device, so a call uploads them with one copy
        sn = steps * n
        nbytes = 8 * sn + 3 * 4 * sn + sn
        self.draws_host = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        self.draws_dev = torch.empty(nbytes, dtype=torch.uint8, device=dev)

        def views(buf):
            u = buf[: 8 * sn].view(torch.float64).view(steps, n)
            i32 = buf[8 * sn: 20 * sn].view(torch.int32).view(3, steps, n)
            return i32[0], buf[20 * sn:].view(steps, n), i32[1], i32[2], u

        self.knob, self.nudge, self.delta, self.resample, self.u = views(self.draws_dev)
        self.host_draws = tuple(t.numpy() for t in views(self.draws_host))
        self.cur = torch.empty((n, nk), dtype=torch.int32, device=dev)
        self.nxt = torch.empty((n, nk), dtype=torch.int32, device=dev)
        self.energy = torch.empty(n, dtype=torch.float64, device=dev)
        self.hist_idx = torch.empty((steps + 1, n), dtype=torch.int64, device=dev)
        self.hist_z = torch.empty((steps + 1, n), dtype=torch.float32, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.temps = []
        t = sched.initial_temp
        for _ in range(steps):
            self.temps.append(t)
            t = max(t * sched.cooling, 1e-9)
        self.graph = None
        import os

        engine = engine or os.environ.get("KT_SA_ENGINE", "fused")
        if engine not in ("fused", "steps"):
            raise DomainError(f"unknown annealing engine {engine!r}")
        self.engine = "fused" if engine == "fused" and n_chains <= 128 else "steps"
        self.temps_dev = torch.tensor(self.temps, dtype=torch.float64, device=dev)
        self.cards_h = np.ascontiguousarray(self.cards_np, dtype=np.int32)
        self.mult_h = np.ascontiguousarray(_space_multipliers(space), dtype=np.int64)

    def _run_fused(self):
        p = _lib.ptr
        _lib.check(self.lib.kt_sa_run(p(self.tab), self.dims, p(self.flat), self.n, self.nk, self.cards_h.ctypes.data,
                                      self.mult_h.ctypes.data, self.sched.steps_per_round, p(self.knob),
                                      p(self.nudge), p(self.delta), p(self.resample), p(self.u), p(self.temps_dev),
                                      p(self.cur), p(self.hist_idx), p(self.hist_z), p(self.err),
                                      _lib.stream_handle(self.dev)), "sa run")

    def _score(self, i, st):
        # after the first score the preceding kernel is kt_sa_propose, which leaves the
        # parameters alone: the scorer may stage its operands under it (PDL)
        p = _lib.ptr
        _lib.check(self.lib.kt_score_indices_flags(p(self.tab), self.dims, p(self.flat), p(self.hist_idx[i]), None, 0,
                                                   self.n, p(self.hist_z[i]), None, None, None, p(self.err),
                                                   1 if i > 0 else 0, st), "sa score")

    def _steps(self):
        p = _lib.ptr
        st = _lib.stream_handle(self.dev)
        self._score(0, st)
        self.energy.copy_(self.hist_z[0].double())
        for s in range(self.sched.steps_per_round):
            _lib.check(self.lib.kt_sa_propose(p(self.cur), self.n, self.nk, p(self.cards), p(self.mult),
                                              p(self.knob[s]), p(self.nudge[s]), p(self.delta[s]),
                                              p(self.resample[s]), p(self.nxt), p(self.hist_idx[s + 1]), st),
                       "sa propose")
            self._score(s + 1, st)
            _lib.check(self.lib.kt_sa_accept(self.n, self.nk, p(self.hist_z[s + 1]), p(self.u[s]), self.temps[s],
                                             p(self.nxt), p(self.cur), p(self.energy), st), "sa accept")

    def explore(self, starts: list, rng) -> dict:
        steps, n = self.sched.steps_per_round, self.n
        knob, nudge, delta, resample, u = self.host_draws
        sa_draws(rng, self.cards_np, knob, nudge, delta, resample, u)
        with torch.cuda.device(self.dev):
            self.draws_dev.copy_(self.draws_host)  # one copy: the five draw arrays are views of one buffer
            start_idx = np.array(starts, dtype=np.int64)
            self.hist_idx[0].copy_(torch.from_numpy(start_idx))
            choices = np.zeros((n, self.nk), dtype=np.int64)
            rest = start_idx.copy()
            for j in range(self.nk - 1, -1, -1):
                choices[:, j] = rest % self.cards_np[j]
                rest //= self.cards_np[j]
            self.cur.copy_(torch.from_numpy(choices.astype(np.int32)))
            if self.engine == "fused":
                self._run_fused()
            elif self.graph is None:
                self._steps()  # eager first run (kernel attributes set outside capture)
                torch.cuda.synchronize(self.dev)
                self.hist_idx[0].copy_(torch.from_numpy(start_idx))
                self.cur.copy_(torch.from_numpy(choices.astype(np.int32)))
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._steps()
                self.graph = g
            if self.engine == "steps":
                self.graph.replay()
            hi = self.hist_idx.cpu().numpy().reshape(-1)
            hz = self.hist_z.cpu().numpy().reshape(-1).astype(np.float64)
        # insertion order: starts, then each step's chains (a revisit keeps its first
        # position and takes the later score, as the reference's dict assignment does)
        return dict(zip(hi.tolist(), hz.tolist()))


_ANNEALERS: dict = {}


def _draws_python(rng, cards, knob, nudge, delta, resample, u) -> None:
    for s in range(knob.shape[0]):  # search.py:233-237, same calls in the same order
        k = rng.integers(0, len(cards), size=knob.shape[1])
        knob[s] = k
        nudge[s] = rng.random(knob.shape[1]) < 0.5
        delta[s] = rng.integers(0, 2, size=knob.shape[1]) * 2 - 1
        resample[s] = rng.integers(0, cards[k])
        u[s] = rng.random(knob.shape[1])


def sa_draws(rng, cards, knob, nudge, delta, resample, u) -> None:
    """Fill the (steps, chains) draw arrays with sa_explore's per-step Generator calls
    (search.py:233-237) and leave `rng` where those calls would leave it.  A PCG64
    Generator (numpy's default, the reference's rng_from) is drawn natively from its
    state (kt_sa_draws, bit-exact with numpy); any other bit generator goes through
    the Generator calls themselves."""
    st = rng.bit_generator.state
    cards = np.asarray(cards, dtype=np.int64)
    if st.get("bit_generator") != "PCG64" or cards.max() >= 2**31:
        _draws_python(rng, cards, knob, nudge, delta, resample, u)
        return
    m64 = (1 << 64) - 1
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    pcg = np.array([s >> 64, s & m64, inc >> 64, inc & m64], dtype=np.uint64)
    has = np.array([st["has_uint32"]], dtype=np.int32)
    ui = np.array([st["uinteger"]], dtype=np.uint32)
    c32 = np.ascontiguousarray(cards, dtype=np.int32)
    for a, dt in ((knob, np.int32), (nudge, np.uint8), (delta, np.int32), (resample, np.int32), (u, np.float64)):
        if a.dtype != dt or not a.flags.c_contiguous or a.shape != knob.shape:
            raise DomainError("sa_draws: draw arrays must be C-contiguous (steps, chains) of the documented dtypes")
    lib = _lib.load()
    p = lambda a: a.ctypes.data  # noqa: E731
    _lib.check(lib.kt_sa_draws(p(pcg), p(has), p(ui), knob.shape[0], knob.shape[1], len(cards), p(c32), p(knob),
                               p(nudge), p(delta), p(resample), p(u)), "sa draws")
    rng.bit_generator.state = {"bit_generator": "PCG64",
                               "state": {"state": (int(pcg[0]) << 64) | int(pcg[1]), "inc": inc},
                               "has_uint32": int(has[0]), "uinteger": int(ui[0])}


def _sa_explore_host(predict, space: KnobSpace, sched: SaSchedule, starts: list, rng) -> dict:
    """The annealing loop on the host for an arbitrary `predict(list[KnobConfig])` callable
    (search.py:202-254; e.g. the reference tune's xgb_energy, search.py:560): the same
    Generator calls in the same order and the same acceptance rule as the device
    annealer, so a shared seed and predictor give the same history."""
    from .kernels import index_config

    cards = np.array(space.cardinalities, dtype=np.int64)
    mult = _space_multipliers(space)
    n = len(starts)
    rows = np.arange(n)
    cur = np.array([index_config(space, i).choices for i in starts], dtype=np.int64).reshape(n, -1)

    def score(mat):
        idx = mat @ mult
        e = np.asarray(predict([index_config(space, int(i)) for i in idx]), dtype=np.float64)
        for i, v in zip(idx.tolist(), e.tolist()):
            history[i] = v
        return e

    history: dict = {}
    energy = score(cur)
    temp = sched.initial_temp
    for _ in range(sched.steps_per_round):
        knob = rng.integers(0, len(cards), size=n)
        nudge = rng.random(n) < 0.5
        delta = rng.integers(0, 2, size=n) * 2 - 1
        resample = rng.integers(0, cards[knob])
        u = rng.random(n)
        nxt = cur.copy()
        nxt[rows, knob] = np.where(nudge, np.clip(cur[rows, knob] + delta, 0, cards[knob] - 1), resample)
        e_new = score(nxt)
        accept = (e_new >= energy) | (u < np.exp(np.minimum((e_new - energy) / temp, 0.0)))
        cur = np.where(accept[:, None], nxt, cur)
        energy = np.where(accept, e_new, energy)
        temp = max(temp * sched.cooling, 1e-9)
    return history


def sa_explore(predict, space: KnobSpace, sched: SaSchedule, visited: set, rng) -> dict:
    """Parallel annealing chains maximizing the cost model (search.py:202-254); returns
    {config_index: score} over everything any chain evaluated, in the reference's
    insertion order.  A CostModelPredictor (default dims, space < 2^32) anneals on the
    device (DeviceAnnealer); any other callable runs the reference-order host loop."""
    starts = draw_unvisited(space, visited, sched.parallel_chains, rng)
    if not starts:
        return {}
    if not (isinstance(predict, CostModelPredictor) and _default_model(predict.m) and space.size < 2**32
            and predict.space == space):
        return _sa_explore_host(predict, space, sched, starts, rng)
    key = (id(predict), sched.initial_temp, sched.cooling, sched.steps_per_round, len(starts))
    ann = _ANNEALERS.get(key)
    # the annealer bakes the parameters and the feature-norm spec table of the predictor's
    # model into its CUDA graph: rebuild when the predictor (or its model) is a new object
    if ann is None or ann.pred is not predict or ann.m is not predict.m:
        if len(_ANNEALERS) > 16:
            _ANNEALERS.clear()
        ann = _ANNEALERS[key] = DeviceAnnealer(predict, sched, len(starts))
    return ann.explore(starts, rng)


def sa_propose(predict, space: KnobSpace, sched: SaSchedule, visited: set, rng, batch: int) -> list:
    """Annealing proposal (search.py:266-281): explore, take the best unvisited configs
    seen, top up with uniform unvisited draws."""
    from .kernels import index_config

    history = sa_explore(predict, space, sched, visited, rng)
    picks = rank_history(history, visited, batch)
    if len(picks) < batch:
        picks += draw_unvisited(space, visited | set(picks), batch - len(picks), rng)
    return [index_config(space, i) for i in picks]


# --- GP surrogate + batch UCB (search.py:39-159, 284-340), the meta-BO proposer ---------------

LENGTHSCALE_GRID = (0.1, 0.3, 1.0, 3.0)  # search.py:37
MAX_JITTER_NOISE = 1e-1                  # search.py:38


@dataclass
class GpSurrogate:
    """search.py:54-66, same fields (host numpy arrays).  The device copies of the
    observations and the factor ride along in `_dev` so predictions do not re-upload."""
    x: np.ndarray
    y: np.ndarray
    lengthscales: np.ndarray | None = None
    noise_variance: float = 1e-4
    chol: np.ndarray | None = None
    alpha: np.ndarray | None = None
    fitted_noise: float | None = None
    _dev: dict | None = None

    @property
    def n_obs(self) -> int:
        return int(self.x.shape[0]) if np.asarray(self.x).ndim == 2 else 0


def knob_coordinates(space: KnobSpace, configs: list) -> np.ndarray:
    """Each knob's value index mapped to [0, 1) by index / cardinality (search.py:65-69)."""
    cards = np.array([len(k.values) for k in space.knobs], dtype=np.float64)
    mat = np.array([c.choices for c in configs], dtype=np.float64).reshape(len(configs), -1)
    return mat / cards


def _d64(a, dev) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(dev)


def _gp_device():
    return torch.device("cuda", torch.cuda.current_device())


def gp_kernel(x1, x2, lengthscales) -> np.ndarray:
    """RBF Gram matrix (search.py:72-76), computed on the device."""
    dev = _gp_device()
    a, b, ls = _d64(x1, dev), _d64(x2, dev), _d64(lengthscales, dev)
    out = torch.empty((a.shape[0], b.shape[0]), dtype=torch.float64, device=dev)
    lib = _lib.load()
    _lib.check(lib.kt_gp_gram(a.data_ptr(), a.shape[0], b.data_ptr(), b.shape[0], a.shape[1], ls.data_ptr(),
                              out.data_ptr(), _lib.stream_handle()), "gp_kernel")
    return out.cpu().numpy()


def gp_fit(s: GpSurrogate, select_lengthscale: bool = True) -> GpSurrogate:
    """Refresh the factorization; optionally pick the isotropic lengthscale by marginal
    likelihood over the grid (search.py:94-121).  All candidates factor concurrently
    (one CTA each, jitter escalation on the device); the first best likelihood wins, and
    a candidate that is not positive definite even at MAX_JITTER_NOISE raises
    NumericError, as the reference does."""
    from dataclasses import replace

    if s.n_obs == 0:
        return s
    x = np.asarray(s.x, dtype=np.float64)
    n, d = x.shape
    if select_lengthscale or s.lengthscales is None:
        cands = np.stack([np.full(d, v) for v in LENGTHSCALE_GRID])
    else:
        cands = np.asarray(s.lengthscales, dtype=np.float64)[None, :]
    dev = _gp_device()
    xd, yd, lsd = _d64(x, dev), _d64(s.y, dev), _d64(cands, dev)
    nc = cands.shape[0]
    L = torch.empty((nc, n, n), dtype=torch.float64, device=dev)
    alpha = torch.empty((nc, n), dtype=torch.float64, device=dev)
    info = torch.empty((nc, 3), dtype=torch.float64, device=dev)
    lib = _lib.load()
    _lib.check(lib.kt_gp_factor(xd.data_ptr(), n, d, lsd.data_ptr(), nc, yd.data_ptr(), float(s.noise_variance),
                                MAX_JITTER_NOISE, L.data_ptr(), alpha.data_ptr(), info.data_ptr(),
                                _lib.stream_handle()), "gp_fit")
    inf = info.cpu().numpy()
    best = None
    for c in range(nc):
        if inf[c, 2] != 0.0:
            raise NumericError(f"kernel matrix not positive definite even at noise {inf[c, 0]:g}")
        if best is None or inf[c, 1] > inf[best, 1]:
            best = c
    Lb = L[best]
    dev_state = {"x": xd, "ls": lsd[best].contiguous(), "L": Lb, "alpha": alpha[best]}
    # the factor is column-major on the device: its host copy's transpose view is the lower L
    return replace(s, lengthscales=cands[best].copy(), chol=Lb.cpu().numpy().T,
                   alpha=alpha[best].cpu().numpy(), fitted_noise=float(inf[best, 0]), _dev=dev_state)


def _require_fitted(s: GpSurrogate) -> None:
    if s.chol is None or s.alpha is None:
        raise DomainError("surrogate not fitted; call gp_fit first")


def _dev_state(s: GpSurrogate) -> dict:
    if s._dev is not None:
        return s._dev
    dev = _gp_device()  # a surrogate fitted elsewhere (e.g. the reference): upload its factor
    return {"x": _d64(s.x, dev), "ls": _d64(s.lengthscales, dev),
            "L": _d64(np.asarray(s.chol).T, dev), "alpha": _d64(s.alpha, dev)}


def _posterior(s: GpSurrogate, xp: np.ndarray, want_cov: bool):
    st = _dev_state(s)
    n, d = st["x"].shape
    dev = st["x"].device
    xpd = _d64(xp, dev)
    P = xpd.shape[0]
    mean = torch.empty(P, dtype=torch.float64, device=dev)
    var = torch.empty(P, dtype=torch.float64, device=dev)
    lib = _lib.load()
    cov = ws = None
    wsb = 0
    if want_cov:
        cov = torch.empty((P, P), dtype=torch.float64, device=dev)
        wsb = int(lib.kt_gp_workspace_bytes(n, P, 0))
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    _lib.check(lib.kt_gp_posterior(st["x"].data_ptr(), n, d, st["ls"].data_ptr(), st["L"].data_ptr(),
                                   st["alpha"].data_ptr(), xpd.data_ptr(), P, mean.data_ptr(), var.data_ptr(),
                                   _lib.ptr(cov), _lib.ptr(ws), wsb, _lib.stream_handle()), "gp posterior")
    return mean, var, cov


def gp_predict_many(s: GpSurrogate, x: np.ndarray) -> tuple:
    """Exact posterior (means, variances) of the latent function (search.py:129-139)."""
    x = np.asarray(x, dtype=np.float64)
    if s.n_obs == 0:
        return np.zeros(x.shape[0]), np.ones(x.shape[0])
    _require_fitted(s)
    mean, var, _ = _posterior(s, x, False)
    return mean.cpu().numpy(), var.cpu().numpy()


def gp_predict(s: GpSurrogate, x) -> tuple:
    mean, var = gp_predict_many(s, np.asarray(x, dtype=np.float64)[None, :])
    return float(mean[0]), float(var[0])


def bo_propose_batch(s: GpSurrogate, space: KnobSpace, batch: int, beta_ucb: float, candidate_pool: int,
                     visited: set, rng, pool: list | None = None) -> list:
    """Sequential UCB over a candidate pool with hallucinated batch downdates
    (search.py:284-340).  Pool construction and RNG draws are the reference's; the
    posterior covariance and the UCB loop run on the device (kt_gp_posterior, kt_gp_ucb)."""
    from .kernels import config_index, index_config

    if batch < 1:
        raise DomainError("batch must be >= 1")
    if pool is None:
        indices = draw_unvisited(space, visited, candidate_pool, rng)
    else:
        seen: set = set()
        indices = []
        for i in configs_to_indices(space, pool).tolist():  # (vectorised config_index)
            if i in visited or i in seen:
                continue
            seen.add(i)
            indices.append(i)
    if not indices:
        raise DomainError("empty candidate pool")
    indices = sorted(indices)
    take = min(batch, len(indices))
    if s.n_obs == 0:
        pick = rng.permutation(len(indices))[:take]
        return [index_config(space, indices[int(i)]) for i in pick]
    _require_fitted(s)
    # knob coordinates straight from the indices (mixed-radix decode, knob 0 most significant)
    cards = np.array([len(k.values) for k in space.knobs], dtype=np.int64)
    rest = np.array(indices, dtype=np.int64)
    ch = np.empty((rest.size, cards.size), dtype=np.float64)
    for j in range(cards.size - 1, -1, -1):
        ch[:, j] = rest % cards[j]
        rest //= cards[j]
    mean, _, cov = _posterior(s, ch / cards, True)
    noise = s.fitted_noise if s.fitted_noise is not None else s.noise_variance
    P = len(indices)
    lib = _lib.load()
    picks = torch.empty(take, dtype=torch.int32, device=mean.device)
    wsb = int(lib.kt_gp_workspace_bytes(0, P, take))
    ws = torch.empty(wsb, dtype=torch.uint8, device=mean.device)
    _lib.check(lib.kt_gp_ucb(mean.data_ptr(), cov.data_ptr(), P, float(noise), float(beta_ucb), take,
                             picks.data_ptr(), ws.data_ptr(), wsb, _lib.stream_handle()), "bo_propose_batch")
    return [index_config(space, indices[int(p)]) for p in picks.cpu().numpy()]
