"""GCN + MLP cost model on the GPU: the drop-in for the reference's model.py.

Same names, signatures and semantics as the reference (kerntune/model.py:54-477):
  ModelState / GcnParams / AggParams / HeadParams / FeatureNorm / LabelNorm /
  Gradients, init_model, normalize_label, denormalize_label, embed_batch,
  head_forward_batch, embed, forward, predict_gflops, loss, grad, sgd_step,
  head_to_vec, vec_to_head, head_loss_grad, head_hvp, save_model, load_model.
Differences, by design:
  * parameters live on the device as fp32 views into ONE flat vector laid out
    [gcn W_i..., agg, head W0, b0, W1, b1, W2, b2] (include/kerntune_b200.h);
    the head part is exactly head_to_vec's order, so MAML/fine-tune update the
    tail of the flat vector in place of the reference's numpy concatenations;
  * FeatureNorm / LabelNorm stay fp64 numpy on the host (they feed the fp64
    encoder tables and the GFLOPS de-normalisation);
  * batch outputs (u, z, gradients) are device tensors; scalars (loss) are
    Python floats, as in the reference.
All compute goes through libkerntune_b200.so; nothing here falls back to CPU.
"""

from __future__ import annotations

import contextlib
import functools
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import DomainError
from .graphs import FEATURE_DIM, tensors_for

LABEL_FLOOR_GFLOPS = 1e-3


@dataclass
class GcnParams:
    layers: list  # (d_in, d_out) fp32 device views


@dataclass
class AggParams:
    sum_weights: torch.Tensor  # (d_last,)


@dataclass
class HeadParams:
    weights: list  # [(2*d_last, h1), (h1, h2), (h2, 1)]
    biases: list


@dataclass
class FeatureNorm:
    mean: np.ndarray
    std: np.ndarray


@dataclass
class LabelNorm:
    mean: float
    std: float


@dataclass
class ModelState:
    gcn: GcnParams
    agg: AggParams
    head: HeadParams
    feature_norm: FeatureNorm
    label_norm: LabelNorm
    _flat: torch.Tensor | None = field(default=None, repr=False, compare=False)


@dataclass
class Gradients:
    gcn: list
    agg: torch.Tensor
    head_weights: list
    head_biases: list
    _flat: torch.Tensor | None = field(default=None, repr=False, compare=False)


# --- layout of the flat parameter vector ---------------------------------------------


_NULL_CTX = contextlib.nullcontext()


def _on(dev):
    """torch.cuda.device(dev), skipped when dev already is the current device."""
    if dev.index is None or dev.index == torch.cuda.current_device():
        return _NULL_CTX
    return torch.cuda.device(dev)


def make_dims(feature_dim: int, gcn_dims, head_hidden) -> _lib.Dims:
    return _make_dims(int(feature_dim), tuple(int(v) for v in gcn_dims), tuple(int(v) for v in head_hidden))


@functools.lru_cache(maxsize=64)
def _make_dims(feature_dim: int, gcn_dims: tuple, head_hidden: tuple) -> _lib.Dims:
    if not gcn_dims or len(gcn_dims) > _lib.KT_MAX_LAYERS or len(head_hidden) + 1 > _lib.KT_MAX_LAYERS + 1:
        raise DomainError("model depth beyond the compiled limits")
    d = _lib.Dims()
    d.F = feature_dim
    d.n_gcn = len(gcn_dims)
    dims = (feature_dim,) + gcn_dims
    for i, v in enumerate(dims):
        d.gcn[i] = v
    off = 0
    for i in range(len(gcn_dims)):
        d.off_gcn[i] = off
        off += dims[i] * dims[i + 1]
    d.off_agg = off
    off += dims[-1]
    hd = (2 * dims[-1],) + head_hidden + (1,)
    d.n_head = len(hd) - 1
    for i, v in enumerate(hd):
        d.head[i] = v
    d.off_head = off
    for i in range(len(hd) - 1):
        d.off_hw[i] = off
        off += hd[i] * hd[i + 1]
        d.off_hb[i] = off
        off += hd[i + 1]
    d.n_head_params = off - d.off_head
    d.n_params = off
    return d


def head_only_dims(head_shapes) -> _lib.Dims:
    """Dims whose offsets index a bare flat head vector (head_to_vec layout)."""
    d = _lib.Dims()
    hd = [head_shapes[0][0]] + [s[1] for s in head_shapes]
    d.n_head = len(head_shapes)
    for i, v in enumerate(hd):
        d.head[i] = v
    off = 0
    for i in range(len(head_shapes)):
        d.off_hw[i] = off
        off += hd[i] * hd[i + 1]
        d.off_hb[i] = off
        off += hd[i + 1]
    d.n_head_params = d.n_params = off
    d.n_gcn = 1
    d.F = d.gcn[0] = d.gcn[1] = 1
    return d


def dims_of(m: ModelState) -> _lib.Dims:
    gcn = [tuple(w.shape) for w in m.gcn.layers]
    return make_dims(gcn[0][0], [s[1] for s in gcn], [w.shape[1] for w in m.head.weights[:-1]])


def _shapes(m) -> list:
    return ([tuple(w.shape) for w in m.gcn.layers] + [tuple(m.agg.sum_weights.shape)]
            + [s for w, b in zip(m.head.weights, m.head.biases) for s in (tuple(w.shape), tuple(b.shape))])


def _tensors(m) -> list:
    return (list(m.gcn.layers) + [m.agg.sum_weights]
            + [t for w, b in zip(m.head.weights, m.head.biases) for t in (w, b)])


def _views(flat: torch.Tensor, shapes: list) -> list:
    out, off = [], 0
    for s in shapes:
        n = int(np.prod(s))
        out.append(flat[off : off + n].view(s))
        off += n
    if off != flat.numel():
        raise DomainError("flat parameter vector has the wrong length")
    return out


def _assemble(cls_state, flat: torch.Tensor, shapes, n_gcn: int, n_head: int, **extra):
    v = _views(flat, shapes)
    gcn, agg, rest = v[:n_gcn], v[n_gcn], v[n_gcn + 1 :]
    hw, hb = rest[0::2], rest[1::2]
    if cls_state is ModelState:
        return ModelState(GcnParams(gcn), AggParams(agg), HeadParams(hw, hb), extra["feature_norm"],
                          extra["label_norm"], _flat=flat)
    return Gradients(gcn=gcn, agg=agg, head_weights=hw, head_biases=hb, _flat=flat)


def _is_packed(obj, tensors) -> bool:
    flat = obj._flat
    if flat is None:
        return False
    base = flat.data_ptr()
    es = flat.element_size()
    off = 0
    for t in tensors:
        if not isinstance(t, torch.Tensor) or t.device != flat.device or t.dtype != flat.dtype:
            return False
        if t.data_ptr() != base + off * es or not t.is_contiguous():
            return False
        off += t.numel()
    return off == flat.numel()


def flat_params(m: ModelState) -> torch.Tensor:
    """The model's flat fp32 device vector; re-packed if the user swapped tensors."""
    ts = _tensors(m)
    if _is_packed(m, ts):
        return m._flat
    dev = m._flat.device if m._flat is not None else _device_of(ts)
    return torch.cat([torch.as_tensor(t, dtype=torch.float32, device=dev).reshape(-1) for t in ts])


def _device_of(ts) -> torch.device:
    for t in ts:
        if isinstance(t, torch.Tensor) and t.is_cuda:
            return t.device
    return torch.device("cuda", torch.cuda.current_device())


def model_from_flat(flat: torch.Tensor, like: ModelState, feature_norm=None, label_norm=None) -> ModelState:
    return _assemble(ModelState, flat, _shapes(like), len(like.gcn.layers), len(like.head.weights),
                     feature_norm=like.feature_norm if feature_norm is None else feature_norm,
                     label_norm=like.label_norm if label_norm is None else label_norm)


def grads_from_flat(flat: torch.Tensor, like: ModelState) -> Gradients:
    return _assemble(Gradients, flat, _shapes(like), len(like.gcn.layers), len(like.head.weights))


def flat_grads(g: Gradients) -> torch.Tensor:
    ts = list(g.gcn) + [g.agg] + [t for w, b in zip(g.head_weights, g.head_biases) for t in (w, b)]
    if _is_packed(g, ts):
        return g._flat
    return torch.cat([torch.as_tensor(t, dtype=torch.float32).reshape(-1) for t in ts])


# --- construction -----------------------------------------------------------------------


def init_model(rng, feature_dim: int = FEATURE_DIM, gcn_dims: tuple = (32, 32),
               head_hidden: tuple = (64, 64), *, device=None) -> ModelState:
    """U(-1/sqrt(fan_in), +) init drawn from `rng` in the reference's order
    (model.py:71-96: gcn layers, then (w_i, b_i) pairs), cast to fp32 on device."""
    def u(fan_in, shape):
        s = 1.0 / math.sqrt(fan_in)
        return rng.uniform(-s, s, size=shape)

    dims = (feature_dim,) + tuple(gcn_dims)
    parts = [u(dims[i], (dims[i], dims[i + 1])) for i in range(len(dims) - 1)]
    parts.append(np.ones(dims[-1]))
    hd = (2 * dims[-1],) + tuple(head_hidden) + (1,)
    for i in range(len(hd) - 1):
        parts.append(u(hd[i], (hd[i], hd[i + 1])))
        parts.append(u(hd[i], (hd[i + 1],)))
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    flat = torch.from_numpy(np.concatenate([p.ravel() for p in parts]).astype(np.float32)).to(dev)
    shapes = [p.shape for p in parts]
    return _assemble(ModelState, flat, shapes, len(gcn_dims), len(hd) - 1,
                     feature_norm=FeatureNorm(np.zeros(feature_dim), np.ones(feature_dim)),
                     label_norm=LabelNorm(0.0, 1.0))


def from_reference(ref_state, *, device=None) -> ModelState:
    """Adopt a reference (numpy fp64) ModelState: same field layout, cast to fp32."""
    parts = (list(ref_state.gcn.layers) + [ref_state.agg.sum_weights]
             + [t for w, b in zip(ref_state.head.weights, ref_state.head.biases) for t in (w, b)])
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    flat = torch.from_numpy(np.concatenate([np.asarray(p).ravel() for p in parts]).astype(np.float32)).to(dev)
    return _assemble(ModelState, flat, [np.asarray(p).shape for p in parts], len(ref_state.gcn.layers),
                     len(ref_state.head.weights),
                     feature_norm=FeatureNorm(np.asarray(ref_state.feature_norm.mean, dtype=np.float64).copy(),
                                              np.asarray(ref_state.feature_norm.std, dtype=np.float64).copy()),
                     label_norm=LabelNorm(float(ref_state.label_norm.mean), float(ref_state.label_norm.std)))


def normalize_label(m: ModelState, gflops: float) -> float:
    return (math.log2(max(gflops, LABEL_FLOOR_GFLOPS)) - m.label_norm.mean) / m.label_norm.std


def denormalize_label(m: ModelState, z):
    """2^(z sigma + mu); works on floats and tensors."""
    if isinstance(z, torch.Tensor):
        return torch.exp2(z.double() * m.label_norm.std + m.label_norm.mean)
    return 2.0 ** (z * m.label_norm.std + m.label_norm.mean)


def loss(preds, labels_normalized) -> float:
    p = np.atleast_1d(np.asarray(_host(preds), dtype=np.float64))
    y = np.atleast_1d(np.asarray(_host(labels_normalized), dtype=np.float64))
    if p.shape != y.shape:
        raise DomainError("prediction/label shape mismatch")
    if p.size == 0:
        raise DomainError("empty batch")
    return float(np.mean((p - y) ** 2))


def _host(x):
    return x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else x


# --- device helpers -----------------------------------------------------------------------

_NORM_CACHE: dict = {}


def _norm_tensors(m: ModelState, dev):
    key = (m.feature_norm.mean.tobytes(), m.feature_norm.std.tobytes(), str(dev))
    hit = _NORM_CACHE.get(key)
    if hit is None:
        hit = (torch.from_numpy(np.asarray(m.feature_norm.mean, dtype=np.float64)).to(dev),
               torch.from_numpy(np.asarray(m.feature_norm.std, dtype=np.float64)).to(dev))
        if len(_NORM_CACHE) > 64:
            _NORM_CACHE.clear()
        _NORM_CACHE[key] = hit
    return hit


_CSR_CACHE: dict = {}


def shared_csr(adj: np.ndarray, dev):
    """CSR (row_ptr, col, fp32 val) of one N x N adjacency, cached per content."""
    adj = np.asarray(adj, dtype=np.float64)
    key = (adj.shape, adj.tobytes(), str(dev))
    hit = _CSR_CACHE.get(key)
    if hit is None:
        rows, cols = np.nonzero(adj)
        row_ptr = np.zeros(adj.shape[0] + 1, dtype=np.int32)
        np.add.at(row_ptr, rows + 1, 1)
        row_ptr = np.cumsum(row_ptr).astype(np.int32)
        hit = (torch.from_numpy(row_ptr).to(dev), torch.from_numpy(cols.astype(np.int32)).to(dev),
               torch.from_numpy(adj[rows, cols].astype(np.float32)).to(dev))
        if len(_CSR_CACHE) > 64:
            _CSR_CACHE.clear()
        _CSR_CACHE[key] = hit
    return hit


def _as_device(x, dev, dtype):
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.dtype(str(dtype).split(".")[-1]))).to(dev)


@dataclass
class PackedGraphs:
    """Segmented-CSR batch of CodeGraphs (device), built by pack_graphs."""
    feats: torch.Tensor      # (total_nodes, F) fp64 raw
    mask: torch.Tensor       # (total_nodes,) uint8
    node_ptr: torch.Tensor   # (B+1,) int64
    row_ptr: torch.Tensor    # (total_nodes+1,) int32
    col: torch.Tensor        # (nnz,) int32 global node ids
    val: torch.Tensor        # (nnz,) fp32
    max_nodes: int
    n_graphs: int


def pack_graphs(graphs, dev) -> PackedGraphs:
    """Host packing of [CodeGraph] into one segmented CSR batch (memoised per graph
    through tensors_for, like the reference's model.py:115-121)."""
    if not graphs:
        raise DomainError("empty batch")
    ts = [tensors_for(g) for g in graphs]
    sizes = np.array([t.feature_matrix.shape[0] for t in ts], dtype=np.int64)
    if sizes.max() > _lib.KT_MAX_NODES:
        raise DomainError(f"graph with {sizes.max()} nodes exceeds the device limit {_lib.KT_MAX_NODES}")
    node_ptr = np.concatenate([[0], np.cumsum(sizes)])
    feats = np.concatenate([t.feature_matrix for t in ts])
    if feats.shape[1] != FEATURE_DIM:
        raise DomainError("feature width mismatch")
    mask = np.concatenate([t.feature_mask for t in ts]).astype(np.uint8)
    rows, cols, vals = [], [], []
    for base, t in zip(node_ptr[:-1], ts):
        r, c = np.nonzero(t.normalized_adjacency)
        rows.append(r + base)
        cols.append(c + base)
        vals.append(t.normalized_adjacency[r, c])
    rows, cols, vals = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    row_ptr = np.zeros(node_ptr[-1] + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    # one staging buffer, one H2D copy, typed device views carved at 16-byte offsets
    parts = [(feats, np.float64), (mask, np.uint8), (node_ptr, np.int64),
             (row_ptr, np.int32), (cols, np.int32), (vals, np.float32)]
    offs, off = [], 0
    for a, dt in parts:
        offs.append(off)
        off += (a.size * np.dtype(dt).itemsize + 15) // 16 * 16
    host = np.empty(max(off, 16), dtype=np.uint8)
    for (a, dt), o in zip(parts, offs):
        n = a.size * np.dtype(dt).itemsize
        host[o:o + n] = np.ascontiguousarray(a, dtype=dt).reshape(-1).view(np.uint8)
    buf = torch.from_numpy(host).to(dev)
    views = []
    for (a, dt), o in zip(parts, offs):
        n = a.size * np.dtype(dt).itemsize
        views.append(buf[o:o + n].view(_TORCH_DT[np.dtype(dt)]).view(a.shape))
    return PackedGraphs(*views, int(sizes.max()), len(graphs))


_TORCH_DT = {np.dtype(np.float64): torch.float64, np.dtype(np.uint8): torch.uint8,
             np.dtype(np.int64): torch.int64, np.dtype(np.int32): torch.int32,
             np.dtype(np.float32): torch.float32}


class _PackedOne:
    """One graph packed in a single device buffer; fields are device addresses
    (embed_graphs only passes pointers), `buf` keeps the allocation alive."""
    __slots__ = ("buf", "feats", "mask", "node_ptr", "row_ptr", "col", "val", "max_nodes", "n_graphs")


def _packed_one(graph, dev):
    """Device pack of one graph, memoised on the graph object per device (the
    single-graph API path: embed / forward / predict_gflops).  Same arrays as
    pack_graphs([graph]), built without the batch concatenations and uploaded
    with one copy."""
    key = str(dev)
    memo = getattr(graph, "_kt_packed", None)
    if memo is not None and memo[0] == key:
        return memo[1]
    t = tensors_for(graph)
    x, adj = t.feature_matrix, t.normalized_adjacency
    n = x.shape[0]
    if n > _lib.KT_MAX_NODES:
        raise DomainError(f"graph with {n} nodes exceeds the device limit {_lib.KT_MAX_NODES}")
    if x.shape[1] != FEATURE_DIM:
        raise DomainError("feature width mismatch")
    nzm = adj != 0
    _, c = np.nonzero(nzm)
    nnz = c.size
    a16 = lambda b: (b + 15) // 16 * 16
    o_mask = a16(x.size * 8)
    o_np = o_mask + a16(n)
    o_rp = o_np + 16
    o_col = o_rp + a16((n + 1) * 4)
    o_val = o_col + a16(nnz * 4)
    host = np.empty(o_val + a16(nnz * 4), dtype=np.uint8)
    host[:x.size * 8].view(np.float64)[:] = x.reshape(-1)
    host[o_mask:o_mask + n] = t.feature_mask
    host[o_np:o_np + 16].view(np.int64)[:] = (0, n)
    rp = host[o_rp:o_rp + (n + 1) * 4].view(np.int32)
    rp[0] = 0
    np.cumsum(np.count_nonzero(nzm, axis=1), out=rp[1:])
    host[o_col:o_col + nnz * 4].view(np.int32)[:] = c
    host[o_val:o_val + nnz * 4].view(np.float32)[:] = adj[nzm]
    pk = _PackedOne()
    pk.buf = torch.from_numpy(host).to(dev)
    base = pk.buf.data_ptr()
    pk.feats, pk.mask, pk.node_ptr = base, base + o_mask, base + o_np
    pk.row_ptr, pk.col, pk.val = base + o_rp, base + o_col, base + o_val
    pk.max_nodes, pk.n_graphs = n, 1
    try:
        graph._kt_packed = (key, pk)
    except AttributeError:
        pass
    return pk


# --- batched forward ----------------------------------------------------------------------


STREAMING_MIN_BATCH = 4096  # embed_batch switches to the streaming layer kernels from here on


def embed_batch(m: ModelState, feats, mask, adj) -> torch.Tensor:
    """Embeddings (B, 2 d) for (B, N, F) raw features sharing one mask/adjacency
    (model.py:185-194); feats may be numpy or a device tensor (e.g. encode_batch's)."""
    flat = flat_params(m)
    dev = flat.device
    x = _as_device(feats, dev, torch.float64)
    if x.dim() != 3 or x.shape[2] != m.gcn.layers[0].shape[0]:
        raise DomainError(f"feats must be (B, N, {m.gcn.layers[0].shape[0]})")
    b, n = x.shape[0], x.shape[1]
    if b == 0:
        raise DomainError("empty batch")
    adj = np.asarray(_host(adj), dtype=np.float64)
    msk = np.asarray(_host(mask), dtype=bool)
    if adj.shape != (n, n) or msk.shape != (n,):
        raise DomainError("adjacency / mask shape does not match feats")
    if n > _lib.KT_MAX_NODES:
        raise DomainError(f"graphs of {n} nodes exceed the device limit {_lib.KT_MAX_NODES}")
    if b >= STREAMING_MIN_BATCH:
        # large batches: the HBM-streaming layer kernels (kt_gcn_layer / kt_readout, ~3.5x the
        # per-graph kernel's throughput at 1M graphs); same results within fp32 rounding
        return embed_batch_streaming(m, x, msk, adj)
    rp, col, val = shared_csr(adj, dev)
    mean, std = _norm_tensors(m, dev)
    mk = torch.from_numpy(msk.astype(np.uint8)).to(dev)
    d = dims_of(m)
    u = torch.empty((b, 2 * d.gcn[d.n_gcn]), dtype=torch.float32, device=dev)
    lib = _lib.load()
    with _on(dev):
        _lib.check(lib.kt_embed_csr(d, _lib.ptr(flat), _lib.ptr(mean), _lib.ptr(std), _lib.ptr(x),
                                    _lib.ptr(mk), None, n, n, _lib.ptr(rp), _lib.ptr(col), _lib.ptr(val), None, b,
                                    _lib.ptr(u), None, _lib.stream_handle()), "embed_batch")
    return u


def head_forward_batch(u, head: HeadParams) -> torch.Tensor:
    """(B,) head outputs (model.py:197-203)."""
    shapes = [tuple(w.shape) for w in head.weights]
    vec = head_to_vec(head)
    dev = vec.device
    uu = _as_device(u, dev, torch.float32)
    if uu.dim() != 2 or uu.shape[1] != shapes[0][0]:
        raise DomainError("u width does not match the head")
    if uu.shape[0] == 0:
        raise DomainError("empty batch")
    z = torch.empty(uu.shape[0], dtype=torch.float32, device=dev)
    lib = _lib.load()
    with _on(dev):
        _lib.check(lib.kt_head_forward(head_only_dims(shapes), _lib.ptr(vec), _lib.ptr(uu), uu.shape[0],
                                       _lib.ptr(z), _lib.stream_handle()), "head_forward_batch")
    return z


def embed_graphs(m: ModelState, graphs, with_scores: bool = False):
    """Embeddings (and optionally scores) of a list of CodeGraphs of any sizes."""
    flat = flat_params(m)
    dev = flat.device
    pk = _packed_one(graphs[0], dev) if len(graphs) == 1 else pack_graphs(graphs, dev)
    mean, std = _norm_tensors(m, dev)
    d = dims_of(m)
    u = torch.empty((pk.n_graphs, 2 * d.gcn[d.n_gcn]), dtype=torch.float32, device=dev)
    z = torch.empty(pk.n_graphs, dtype=torch.float32, device=dev) if with_scores else None
    lib = _lib.load()
    with _on(dev):
        _lib.check(lib.kt_embed_csr(d, _lib.ptr(flat), _lib.ptr(mean), _lib.ptr(std), _lib.ptr(pk.feats),
                                    _lib.ptr(pk.mask), _lib.ptr(pk.node_ptr), 0, pk.max_nodes,
                                    _lib.ptr(pk.row_ptr), _lib.ptr(pk.col), _lib.ptr(pk.val), None, pk.n_graphs,
                                    _lib.ptr(u), _lib.ptr(z), _lib.stream_handle()), "embed_graphs")
    return (u, z) if with_scores else u


# --- streaming layer path: the HBM-bound aggregation kernels -------------------------------


@dataclass
class AdjPatterns:
    """Distinct normalised adjacencies of a batch as local CSRs (kt_gcn_layer's input)."""
    n_pat: int
    pat_n: torch.Tensor     # (n_pat,) int32 nodes per pattern
    rp: torch.Tensor        # concatenated local row_ptr, (n + 1) per pattern
    col: torch.Tensor       # concatenated local column ids
    val: torch.Tensor       # fp32 of the fp64 A_hat entries
    mask: torch.Tensor      # concatenated node masks (uint8)
    nnz: int
    max_nodes: int


_PAT_CACHE: dict = {}


def adjacency_patterns(adjs, masks, dev) -> AdjPatterns:
    """Local CSR (row-major nonzeros of the fp64 A_hat, graphs.py:234-241) of each
    distinct adjacency, cached by content."""
    adjs = [np.asarray(_host(a), dtype=np.float64) for a in adjs]
    masks = [np.asarray(_host(mk), dtype=bool) for mk in masks]
    key = (tuple(a.tobytes() for a in adjs), tuple(mk.tobytes() for mk in masks), str(dev))
    hit = _PAT_CACHE.get(key)
    if hit is not None:
        return hit
    if len(adjs) > 8:
        raise DomainError("kt_gcn_layer takes at most 8 distinct adjacency patterns per batch")
    rps, cols, vals, mks, ns = [], [], [], [], []
    for a, mk in zip(adjs, masks):
        if a.shape[0] > _lib.KT_MAX_NODES:
            raise DomainError(f"graphs of {a.shape[0]} nodes exceed the device limit {_lib.KT_MAX_NODES}")
        r, c = np.nonzero(a)
        rp = np.zeros(a.shape[0] + 1, dtype=np.int64)
        np.add.at(rp, r + 1, 1)
        rps.append(np.cumsum(rp))
        cols.append(c)
        vals.append(a[r, c])
        mks.append(mk.astype(np.uint8))
        ns.append(a.shape[0])
    nnz = int(sum(len(c) for c in cols))
    if nnz > 1024:
        raise DomainError("kt_gcn_layer takes at most 1024 adjacency nonzeros per batch")
    up = lambda x, dt: torch.from_numpy(np.ascontiguousarray(np.concatenate(x), dtype=dt)).to(dev)
    hit = AdjPatterns(len(adjs), torch.tensor(ns, dtype=torch.int32, device=dev), up(rps, np.int32),
                      up(cols, np.int32), up(vals, np.float32), up(mks, np.uint8), nnz, int(max(ns)))
    if len(_PAT_CACHE) > 64:
        _PAT_CACHE.clear()
    _PAT_CACHE[key] = hit
    return hit


def _gcn_layers(m: ModelState, x64: torch.Tensor, n_graphs: int, n_uniform: int, node_ptr, pat_id,
                pats: AdjPatterns) -> torch.Tensor:
    """All GCN layers through kt_gcn_layer: fp64 raw rows in, fp32 H_L rows out."""
    flat = flat_params(m)
    dev = flat.device
    mean, std = _norm_tensors(m, dev)
    rows = x64.shape[0]
    lib = _lib.load()
    h = x64
    for i, w in enumerate(m.gcn.layers):
        d_in, d_out = int(w.shape[0]), int(w.shape[1])
        if h.shape[1] != d_in:
            raise DomainError(f"GCN input width {h.shape[1]} != weight rows {d_in}")
        out = torch.empty((rows, d_out), dtype=torch.float32, device=dev)
        wc = w.contiguous()
        with _on(dev):
            _lib.check(lib.kt_gcn_layer(_lib.ptr(h), int(i == 0), _lib.ptr(mean), _lib.ptr(std), _lib.ptr(wc),
                                        d_in, d_out, 1, n_graphs, n_uniform, _lib.ptr(node_ptr), _lib.ptr(pat_id),
                                        pats.n_pat, _lib.ptr(pats.pat_n), _lib.ptr(pats.rp), _lib.ptr(pats.col),
                                        _lib.ptr(pats.val), _lib.ptr(pats.mask), pats.nnz, pats.max_nodes,
                                        _lib.ptr(out), _lib.stream_handle()), "gcn_layer")
        h = out
    return h


def gcn_forward_batch(m: ModelState, feats, mask, adj) -> torch.Tensor:
    """gcn_forward (model.py:127-133) for a batch sharing one adjacency / mask:
    (B, N, F) raw features -> H_L (B, N, d_L) fp32, one streaming kernel per layer."""
    dev = flat_params(m).device
    x = _as_device(feats, dev, torch.float64)
    if x.dim() != 3 or x.shape[2] != m.gcn.layers[0].shape[0]:
        raise DomainError(f"feats must be (B, N, {m.gcn.layers[0].shape[0]})")
    b, n = x.shape[0], x.shape[1]
    if b == 0:
        raise DomainError("empty batch")
    adj = np.asarray(_host(adj), dtype=np.float64)
    msk = np.asarray(_host(mask), dtype=bool)
    if adj.shape != (n, n) or msk.shape != (n,):
        raise DomainError("adjacency / mask shape does not match feats")
    pats = adjacency_patterns([adj], [msk], dev)
    h = _gcn_layers(m, x.reshape(b * n, -1), b, n, None, None, pats)
    return h.reshape(b, n, -1)


def gcn_forward_graphs(m: ModelState, graphs):
    """gcn_forward over CodeGraphs of any sizes: H_L rows (total nodes, d_L) and the
    int64 node_ptr (B + 1) segmenting them."""
    if not graphs:
        raise DomainError("empty batch")
    dev = flat_params(m).device
    ts = [tensors_for(g) for g in graphs]
    keys, pat_of, adjs, masks = {}, [], [], []
    for t in ts:
        k = (t.normalized_adjacency.tobytes(), np.asarray(t.feature_mask).tobytes())
        if k not in keys:
            keys[k] = len(adjs)
            adjs.append(t.normalized_adjacency)
            masks.append(t.feature_mask)
        pat_of.append(keys[k])
    pats = adjacency_patterns(adjs, masks, dev)
    sizes = np.array([t.feature_matrix.shape[0] for t in ts], dtype=np.int64)
    node_ptr = torch.from_numpy(np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)).to(dev)
    x = torch.from_numpy(np.ascontiguousarray(np.concatenate([t.feature_matrix for t in ts]),
                                              dtype=np.float64)).to(dev)
    pid = torch.tensor(pat_of, dtype=torch.int32, device=dev)
    return _gcn_layers(m, x, len(graphs), 0, node_ptr, pid, pats), node_ptr


def aggregate_batch(h, agg: AggParams, node_ptr=None) -> torch.Tensor:
    """aggregate (model.py:136-141) per graph: h (B, N, d) -> (B, 2 d); or h (rows, d)
    segmented by node_ptr (B + 1).  Warp-shuffle segmented reductions (kt_readout)."""
    w = agg.sum_weights
    dev = w.device
    hh = _as_device(h, dev, torch.float32)
    d = int(w.shape[0])
    if hh.shape[-1] != d:
        raise DomainError("embedding width does not match aggregation weights")
    if node_ptr is None:
        if hh.dim() != 3 or hh.shape[0] == 0 or hh.shape[1] == 0:
            raise DomainError("cannot aggregate an empty embedding matrix")
        b, n = hh.shape[0], hh.shape[1]
        np_t = None
    else:
        np_t = _as_device(node_ptr, dev, torch.int64)
        b, n = np_t.numel() - 1, 0
        if b <= 0:
            raise DomainError("empty batch")
    u = torch.empty((b, 2 * d), dtype=torch.float32, device=dev)
    wc = w.contiguous()  # (held: a bare pointer to a temporary could be reallocated before the launch)
    lib = _lib.load()
    with _on(dev):
        _lib.check(lib.kt_readout(_lib.ptr(hh), d, b, n, _lib.ptr(np_t), _lib.ptr(wc), _lib.ptr(u),
                                  _lib.stream_handle()), "aggregate_batch")
    return u


def embed_batch_streaming(m: ModelState, feats, mask, adj) -> torch.Tensor:
    """embed_batch (model.py:185-194) as layer kernels + readout: same result as
    embed_batch, materialising H_l in HBM (the form large batches stream through)."""
    return aggregate_batch(gcn_forward_batch(m, feats, mask, adj), m.agg)


def embed(graph, m: ModelState) -> torch.Tensor:
    """Aggregated embedding of one graph (model.py:153-160)."""
    return embed_graphs(m, [graph])[0]


def forward(graph, m: ModelState) -> float:
    """Prediction on the normalised log scale (model.py:163-165)."""
    return float(embed_graphs(m, [graph], with_scores=True)[1][0].item())


def predict_gflops(graph, m: ModelState) -> float:
    return denormalize_label(m, forward(graph, m))


# --- flat head parameterisation (model.py:328-355) -------------------------------------------


def head_to_vec(head: HeadParams) -> torch.Tensor:
    """Flat [W0, b0, W1, b1, ...] vector; a view when the head already is one."""
    parts = [t for w, b in zip(head.weights, head.biases) for t in (w, b)]
    if all(isinstance(t, torch.Tensor) for t in parts):
        base, off, ok = parts[0], 0, True
        for t in parts:
            if (not t.is_contiguous() or t.dtype != base.dtype or t.device != base.device
                    or t.data_ptr() != base.data_ptr() + off * base.element_size()):
                ok = False
                break
            off += t.numel()
        if ok:
            return torch.as_strided(base, (off,), (1,))
    dev = _device_of(parts)
    return torch.cat([torch.as_tensor(t, dtype=torch.float32, device=dev).reshape(-1) for t in parts])


def vec_to_head(vec, like: HeadParams) -> HeadParams:
    vec = torch.as_tensor(vec)
    ws, bs, off = [], [], 0
    for w, b in zip(like.weights, like.biases):
        nw, nb = int(np.prod(w.shape)), int(np.prod(b.shape))
        ws.append(vec[off : off + nw].view(tuple(w.shape)))
        off += nw
        bs.append(vec[off : off + nb].view(tuple(b.shape)))
        off += nb
    if off != vec.numel():
        raise DomainError("flat head vector has the wrong length")
    return HeadParams(weights=ws, biases=bs)


def with_head_vec(m: ModelState, head_vec: torch.Tensor) -> ModelState:
    """New ModelState sharing gcn/agg values with m and taking `head_vec` as its head."""
    d = dims_of(m)
    flat = flat_params(m)
    new = torch.cat([flat[: d.off_head], head_vec.reshape(-1).to(flat.dtype)])
    return model_from_flat(new, m)


# --- gradients and SGD (model.py:218-310) --------------------------------------------------


def _grad_packed(m: ModelState, pk: PackedGraphs, y: torch.Tensor, scope: str, graph_idx=None, *,
                 lr: float | None = None, npg: int = 0):
    """Device grad over a packed batch; returns (loss tensor fp64 (1,), grad flat, new flat or None)."""
    if scope not in ("all", "head_only"):
        raise DomainError(f"unknown grad scope {scope!r}")
    flat = flat_params(m)
    dev = flat.device
    d = dims_of(m)
    b = int(graph_idx.numel()) if graph_idx is not None else pk.n_graphs
    if b == 0:
        raise DomainError("empty batch")
    mean, std = _norm_tensors(m, dev)
    lib = _lib.load()
    ws_bytes = int(lib.kt_grad_workspace_bytes(d, b))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    g = torch.empty_like(flat)
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    new = torch.empty_like(flat) if lr is not None else None
    with _on(dev):
        _lib.check(lib.kt_grad(d, _lib.ptr(flat), _lib.ptr(mean), _lib.ptr(std), _lib.ptr(pk.feats),
                               _lib.ptr(pk.mask), None if npg else _lib.ptr(pk.node_ptr), npg, pk.max_nodes,
                               _lib.ptr(pk.row_ptr), _lib.ptr(pk.col), _lib.ptr(pk.val), _lib.ptr(graph_idx),
                               _lib.ptr(y), b, 1 if scope == "head_only" else 0, _lib.ptr(g), _lib.ptr(loss),
                               0.0 if lr is None else float(lr), _lib.ptr(new), _lib.ptr(ws), ws_bytes,
                               _lib.stream_handle()), "grad")
    return loss, g, new


def grad(m: ModelState, batch: list, scope: str = "all"):
    """(loss, Gradients) of the batch MSE over [(graph, label_gflops)] (model.py:218-285).

    scope "head_only" leaves gcn/agg gradients exactly zero."""
    if scope not in ("all", "head_only"):
        raise DomainError(f"unknown grad scope {scope!r}")
    if not batch:
        raise DomainError("empty batch")
    ys = np.array([normalize_label(m, float(v)) for _, v in batch], dtype=np.float64)
    if not np.isfinite(ys).all():
        raise DomainError("non-finite label")
    dev = flat_params(m).device
    pk = pack_graphs([g for g, _ in batch], dev)
    y = torch.from_numpy(ys.astype(np.float32)).to(dev)
    loss, g, _ = _grad_packed(m, pk, y, scope)
    return float(loss.item()), grads_from_flat(g, m)


def _sgd_flat(p: torch.Tensor, g: torch.Tensor, lr: float) -> torch.Tensor:
    if p.shape != g.shape:
        raise DomainError("parameter/gradient shape mismatch")
    pc = p.contiguous().float()
    gc = g.to(device=pc.device, dtype=torch.float32).contiguous()
    out = torch.empty_like(pc)
    if pc.numel() == 0:
        return out
    lib = _lib.load()
    with torch.cuda.device(pc.device):
        _lib.check(lib.kt_sgd(_lib.ptr(pc), _lib.ptr(gc), float(lr), pc.numel(), _lib.ptr(out),
                              _lib.stream_handle()), "sgd_step")
    return out


def sgd_step(p, g, lr: float):
    """p - lr*g for ModelState/Gradients, HeadParams/Gradients or plain arrays (model.py:288-310)."""
    if isinstance(p, ModelState) and isinstance(g, Gradients):
        if _shapes(p) != [tuple(t.shape) for t in
                          list(g.gcn) + [g.agg] + [t for w, b in zip(g.head_weights, g.head_biases) for t in (w, b)]]:
            raise DomainError("gradient shapes do not match parameters")
        return model_from_flat(_sgd_flat(flat_params(p), flat_grads(g), lr), p)
    if isinstance(p, HeadParams) and isinstance(g, Gradients):
        gh = HeadParams(list(g.head_weights), list(g.head_biases))
        return vec_to_head(_sgd_flat(head_to_vec(p), head_to_vec(gh), lr), p)
    if isinstance(p, (np.ndarray, torch.Tensor)) and isinstance(g, (np.ndarray, torch.Tensor)):
        if tuple(p.shape) != tuple(g.shape):
            raise DomainError("parameter/gradient shape mismatch")
        was_np = isinstance(p, np.ndarray)
        dev = p.device if isinstance(p, torch.Tensor) and p.is_cuda else torch.device("cuda", torch.cuda.current_device())
        pt = torch.as_tensor(p, dtype=torch.float32).to(dev).reshape(-1)
        out = _sgd_flat(pt, torch.as_tensor(g, dtype=torch.float32).to(dev).reshape(-1), lr).view(tuple(p.shape))
        return out.cpu().numpy().astype(p.dtype) if was_np else out
    raise DomainError(f"cannot apply sgd_step to {type(p).__name__}/{type(g).__name__}")


# --- head engine on flat vectors (model.py:358-432) ------------------------------------------


def _head_dims_like(like: HeadParams) -> _lib.Dims:
    return head_only_dims([tuple(w.shape) for w in like.weights])


def _dev_vec(x, dev):
    return torch.as_tensor(x, dtype=torch.float32).to(dev).contiguous().reshape(-1)


def head_loss_grad(vec, like: HeadParams, u, y):
    """(mse, d mse / d vec) of the head at flat params `vec` on embeddings u (n, D)."""
    d = _head_dims_like(like)
    dev = _device_of([vec] + list(like.weights))
    v = _dev_vec(vec, dev)
    if v.numel() != d.n_head_params:
        raise DomainError("flat head vector has the wrong length")
    uu = torch.as_tensor(u, dtype=torch.float32).to(dev).contiguous()
    yy = _dev_vec(y, dev)
    if uu.dim() != 2 or uu.shape[1] != d.head[0] or uu.shape[0] != yy.numel():
        raise DomainError("u / y shapes do not match the head")
    g = torch.empty_like(v)
    mse = torch.empty(1, dtype=torch.float32, device=dev)
    lib = _lib.load()
    with _on(dev):
        _lib.check(lib.kt_head_loss_grad(d, _lib.ptr(v), _lib.ptr(uu), _lib.ptr(yy), uu.shape[0], _lib.ptr(g),
                                         _lib.ptr(mse), _lib.stream_handle()), "head_loss_grad")
    return float(mse.item()), g


def head_hvp(vec, like: HeadParams, u, y, v) -> torch.Tensor:
    """Hessian-vector product of the head MSE at `vec` along `v` (forward-over-reverse)."""
    d = _head_dims_like(like)
    dev = _device_of([vec] + list(like.weights))
    th = _dev_vec(vec, dev)
    vv = _dev_vec(v, dev)
    if th.numel() != d.n_head_params or vv.numel() != d.n_head_params:
        raise DomainError("flat head vector has the wrong length")
    uu = torch.as_tensor(u, dtype=torch.float32).to(dev).contiguous()
    yy = _dev_vec(y, dev)
    out = torch.empty_like(th)
    lib = _lib.load()
    with _on(dev):
        _lib.check(lib.kt_head_hvp(d, _lib.ptr(th), _lib.ptr(uu), _lib.ptr(yy), _lib.ptr(vv), uu.shape[0],
                                   _lib.ptr(out), _lib.stream_handle()), "head_hvp")
    return out


# --- checkpoints (model.py:438-477, npz v1) ----------------------------------------------------

CHECKPOINT_VERSION = 1


def save_model(m: ModelState, path) -> None:
    """npz v1, interchangeable with the reference; fp32 weights are stored as fp64."""
    h = lambda t: np.asarray(_host(t), dtype=np.float64)
    arrays = {
        "version": np.array(CHECKPOINT_VERSION),
        "n_gcn": np.array(len(m.gcn.layers)),
        "agg_w": h(m.agg.sum_weights),
        "feat_mean": np.asarray(m.feature_norm.mean, dtype=np.float64),
        "feat_std": np.asarray(m.feature_norm.std, dtype=np.float64),
        "label_norm": np.array([m.label_norm.mean, m.label_norm.std]),
    }
    for i, w in enumerate(m.gcn.layers):
        arrays[f"gcn_{i}"] = h(w)
    for i, (w, b) in enumerate(zip(m.head.weights, m.head.biases)):
        arrays[f"head_w{i}"] = h(w)
        arrays[f"head_b{i}"] = h(b)
    np.savez(path, **arrays)


def load_model(path, *, device=None) -> ModelState:
    with np.load(path) as z:
        if int(z["version"]) != CHECKPOINT_VERSION:
            raise DomainError(f"unsupported checkpoint version {int(z['version'])}")
        n_gcn = int(z["n_gcn"])
        parts = [z[f"gcn_{i}"] for i in range(n_gcn)] + [z["agg_w"]]
        i = 0
        while f"head_w{i}" in z:
            parts += [z[f"head_w{i}"], z[f"head_b{i}"]]
            i += 1
        label = z["label_norm"]
        fn = FeatureNorm(z["feat_mean"].copy(), z["feat_std"].copy())
        ln = LabelNorm(float(label[0]), float(label[1]))
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    flat = torch.from_numpy(np.concatenate([p.ravel() for p in parts]).astype(np.float32)).to(dev)
    return _assemble(ModelState, flat, [p.shape for p in parts], n_gcn, i, feature_norm=fn, label_norm=ln)
