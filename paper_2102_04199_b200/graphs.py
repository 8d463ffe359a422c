"""Schedule graphs, super-graph template, batch layouts, and the device encoder.

Host side (once per spec / per graph object):
  * the star-shaped loop graph and the super-graph template
    (reference graphs.py:30-228),
  * the symmetric-normalised adjacency D^-1/2 (A+I) D^-1/2 built in fp64
    exactly as reference graphs.py:234-241,
  * `batch_layout` (graphs.py:278-302), and
  * `EncodeTables`: the per-spec constants the device encoder needs.

Device side (per candidate): `encode_batch` (graphs.py:305-351) runs as the
sm_100a kernel `kt_encode` -- index/choice decode, clamp + ceil-split, the 12
context slots, scatter into iterval rows -- and returns a device tensor.
"""

from __future__ import annotations

import ctypes
import operator
from dataclasses import dataclass

import numpy as np

from .errors import DomainError
from .kernels import (
    AXES_BY_OP,
    AXIS_ORDER,
    KEY_SHIFT,
    MAX_KNOBS,
    REDUCTION_AXES,
    KernelSpec,
    KnobConfig,
    KnobSpace,
    axis_extents,
    build_knob_space,
    card_code,
    knob_value_map,
    resolved_tiles,
)

FEATURE_SLOTS = (
    "extent",
    "log2_extent",
    "tile_level",
    "is_reduction",
    "is_unrolled",
    "stride_hint",
    "touched_elements_estimate",
    "log2_touched",
    "arithmetic_ops_estimate",
    "log2_arith",
    "loop_depth",
    "normalized_position",
)
FEATURE_DIM = len(FEATURE_SLOTS)


@dataclass
class GraphNode:
    kind: str  # "root" | "for_node" | "iterval"
    feature: np.ndarray | None = None
    template_slot: str | None = None


@dataclass
class CodeGraph:
    nodes: list
    edges: list
    label: float | None = None

    @property
    def num_nodes(self) -> int:
        return len(self.nodes)


@dataclass(frozen=True)
class SuperGraphTemplate:
    op_types: tuple
    slots: tuple
    mapping_table: dict

    @property
    def num_nodes(self) -> int:
        return 1 + 2 * len(self.slots)

    def iterval_index(self, slot: str) -> int:
        return 2 + 2 * self.slots.index(slot)


@dataclass
class GraphTensors:
    feature_matrix: np.ndarray  # (N, F) fp64, raw (unnormalised)
    normalized_adjacency: np.ndarray  # (N, N) fp64
    feature_mask: np.ndarray  # (N,) bool


# --- loop context features (host fp64; used for CodeGraph construction) -------


def context_features(extents, tile_levels, reductions, unrolled, stride_hints) -> np.ndarray:
    """12 feature slots per loop; last axis = loops outermost-first (graphs.py:89-126).

    touched = product of the extents strictly inside a loop; arith = 2*touched;
    logs are log2(max(v, 1)); depth = 1..n; position = k / max(n-1, 1).
    """
    e = np.asarray(extents, dtype=np.float64)
    n = e.shape[-1]
    touched = np.ones_like(e)
    if n > 1:
        suffix = np.cumprod(e[..., ::-1], axis=-1)[..., ::-1]
        touched[..., :-1] = suffix[..., 1:]
    arith = 2.0 * touched
    lg = lambda v: np.log2(np.maximum(v, 1.0))
    depth = np.broadcast_to(np.arange(1, n + 1, dtype=np.float64), e.shape)
    pos = np.broadcast_to(np.arange(n, dtype=np.float64) / max(n - 1, 1), e.shape)
    cols = [e, lg(e), tile_levels, reductions, unrolled, stride_hints,
            touched, lg(touched), arith, lg(arith), depth, pos]
    cols = [np.asarray(c, dtype=np.float64) for c in cols]
    return np.stack(np.broadcast_arrays(*cols), axis=-1)


def loop_slot_names(axes) -> list:
    """Chain order of the lowered nest: all outer loops, then all inner loops."""
    present = set(axes)
    return [f"{a}_{s}" for s in ("outer", "inner") for a in AXIS_ORDER if a in present]


def _loop_rows(spec: KernelSpec, space: KnobSpace, config: KnobConfig):
    values = knob_value_map(space, config)
    tiles = resolved_tiles(spec, values)
    auto = int(values.get("auto_unroll_max_step", 0))
    explicit = bool(values.get("unroll_explicit", 0))
    axes = AXES_BY_OP[spec.op_type]
    ext, lvl, red, unr, strd = [], [], [], [], []
    for level in (0, 1):
        for a in axes:
            outer, inner = tiles[a]
            e = outer if level == 0 else inner
            ext.append(e)
            lvl.append(level)
            red.append(1.0 if a in REDUCTION_AXES else 0.0)
            unr.append(1.0 if (level == 1 and explicit and 0 < e <= auto) else 0.0)
            strd.append(float(inner) if level == 0 else 1.0)
    return loop_slot_names(axes), context_features(ext, lvl, red, unr, strd)


# --- templates and graphs -------------------------------------------------------


def build_super_template(op_types) -> SuperGraphTemplate:
    ops = tuple(sorted(set(op_types)))
    if not ops:
        raise DomainError("op_types must be non-empty")
    for op in ops:
        if op not in AXES_BY_OP:
            raise DomainError(f"unsupported op_type {op!r}")
    union = set()
    for op in ops:
        union.update(AXES_BY_OP[op])
    slots = tuple(loop_slot_names(union))
    mapping = {(op, name): name for op in ops for name in loop_slot_names(AXES_BY_OP[op])}
    return SuperGraphTemplate(op_types=ops, slots=slots, mapping_table=mapping)


def _star(names, features=None):
    nodes, edges = [GraphNode("root")], []
    for i, name in enumerate(names):
        f = len(nodes)
        nodes.append(GraphNode("for_node", template_slot=name))
        feat = None if features is None or features[i] is None else np.array(features[i])
        nodes.append(GraphNode("iterval", feature=feat, template_slot=name))
        edges += [(0, f), (f, f + 1)]
    return nodes, edges


def template_graph_skeleton(template: SuperGraphTemplate) -> CodeGraph:
    nodes, edges = _star(template.slots)
    return CodeGraph(nodes=nodes, edges=edges)


def augment_to_super(graph: CodeGraph, template: SuperGraphTemplate, op_type: str) -> CodeGraph:
    out = template_graph_skeleton(template)
    out.label = graph.label
    for node in graph.nodes:
        if node.kind != "iterval":
            continue
        slot = template.mapping_table.get((op_type, node.template_slot))
        if slot is None:
            raise DomainError(f"template has no slot for {(op_type, node.template_slot)}")
        if node.feature is not None:
            out.nodes[template.iterval_index(slot)].feature = node.feature.copy()
    return out


def config_graph(spec, config, space=None, template=None, label=None) -> CodeGraph:
    """Star graph of (spec, config): root -> for_node -> iterval per loop,
    optionally augmented into `template` (reference graphs.py:354-369)."""
    if space is None:
        space = build_knob_space(spec)
    names, feats = _loop_rows(spec, space, config)
    nodes, edges = _star(names, list(feats))
    g = CodeGraph(nodes=nodes, edges=edges, label=label)
    if template is not None:
        g = augment_to_super(g, template, spec.op_type)
    return g


def feature_multiset(graph: CodeGraph) -> list:
    return sorted(tuple(n.feature.tolist()) for n in graph.nodes if n.feature is not None)


# --- tensorisation ------------------------------------------------------------------


def normalized_adjacency(num_nodes: int, edges) -> np.ndarray:
    """D^-1/2 (A + I) D^-1/2 in fp64, same operation order as graphs.py:234-241."""
    a = np.zeros((num_nodes, num_nodes))
    if len(edges):
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        a[e[:, 0], e[:, 1]] = 1.0
        a[e[:, 1], e[:, 0]] = 1.0
    a[np.diag_indices(num_nodes)] += 1.0
    dinv = 1.0 / np.sqrt(a.sum(axis=1))
    return a * dinv[:, None] * dinv[None, :]


def graph_to_tensors(graph) -> GraphTensors:
    n = len(graph.nodes)
    x = np.zeros((n, FEATURE_DIM))
    mask = np.zeros(n, dtype=bool)
    for i, node in enumerate(graph.nodes):
        if node.feature is None:
            continue
        f = np.asarray(node.feature)
        if f.shape != (FEATURE_DIM,):
            raise DomainError(f"node {i} feature has shape {f.shape}, want ({FEATURE_DIM},)")
        x[i] = f
        mask[i] = True
    return GraphTensors(x, normalized_adjacency(n, graph.edges), mask)


def tensors_for(graph) -> GraphTensors:
    """Memoised graph_to_tensors (reference model.py:115-121 memoises the same way)."""
    cached = getattr(graph, "_tensors", None)
    if cached is None:
        cached = graph_to_tensors(graph)
        graph._tensors = cached
    return cached


@dataclass
class BatchLayout:
    adjacency: np.ndarray
    iterval_rows: np.ndarray
    feature_mask: np.ndarray
    num_nodes: int
    loop_names: tuple


def batch_layout(spec: KernelSpec, template: SuperGraphTemplate | None) -> BatchLayout:
    """Shared adjacency / iterval rows / mask for a spec (graphs.py:278-302)."""
    names = loop_slot_names(AXES_BY_OP[spec.op_type])
    if template is None:
        rows = np.array([2 + 2 * i for i in range(len(names))])
        nodes, edges = _star(names)
    else:
        rows = np.array([template.iterval_index(template.mapping_table[(spec.op_type, n)])
                         for n in names])
        nodes, edges = _star(template.slots)
    num = len(nodes)
    mask = np.zeros(num, dtype=bool)
    mask[rows] = True
    return BatchLayout(normalized_adjacency(num, edges), rows, mask, num, tuple(names))


# --- text format (reference graphs.py:381-429) -----------------------------------


def graph_to_text(graph: CodeGraph) -> str:
    lines = [f"codegraph {graph.num_nodes} {FEATURE_DIM}"]
    for n in graph.nodes:
        slot = n.template_slot if n.template_slot is not None else "-"
        body = "null" if n.feature is None else " ".join(repr(float(v)) for v in n.feature)
        lines.append(f"{n.kind} {slot} {body}")
    lines += [f"edge {s} {d}" for s, d in graph.edges]
    if graph.label is not None:
        lines.append(f"label {repr(float(graph.label))}")
    return "\n".join(lines) + "\n"


def graph_from_text(text: str) -> CodeGraph:
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines or not lines[0].startswith("codegraph "):
        raise DomainError("not a codegraph document")
    _, n_s, f_s = lines[0].split()[:3]
    num_nodes = int(n_s)
    if int(f_s) != FEATURE_DIM:
        raise DomainError(f"feature dim {f_s} unsupported (want {FEATURE_DIM})")
    if len(lines) < 1 + num_nodes:
        raise DomainError("truncated codegraph document")
    nodes = []
    for ln in lines[1 : 1 + num_nodes]:
        kind, slot, *rest = ln.split()
        slot = None if slot == "-" else slot
        if rest == ["null"]:
            nodes.append(GraphNode(kind, template_slot=slot))
            continue
        vals = np.array([float(v) for v in rest])
        if vals.shape != (FEATURE_DIM,):
            raise DomainError("bad feature row length")
        nodes.append(GraphNode(kind, feature=vals, template_slot=slot))
    edges, label = [], None
    for ln in lines[1 + num_nodes :]:
        parts = ln.split()
        if parts[0] == "edge":
            edges.append((int(parts[1]), int(parts[2])))
        elif parts[0] == "label":
            label = float(parts[1])
        else:
            raise DomainError(f"unexpected line {ln!r}")
    return CodeGraph(nodes=nodes, edges=edges, label=label)


# --- device encode tables ----------------------------------------------------------


def _norm32(x, mean, std, slot):
    """np.float32((x - mean[slot]) / std[slot]) in fp64 -- the reference's order
    of operations (model.py:111), so table entries are bit-exact."""
    return np.float32((np.float64(x) - mean[slot]) / std[slot])


def build_spec_table(spec: KernelSpec, space: KnobSpace, layout: BatchLayout,
                     fmean=None, fstd=None):
    """Host-side `kt_spec_table` for (spec, space, layout, feature norm).

    Everything that depends on a single tile choice or only on the loop
    position is tabulated here with numpy fp64 (so it is bit-identical to
    encode_batch + normalize_features); the device computes the rest.
    """
    from . import _lib

    fmean = np.zeros(FEATURE_DIM) if fmean is None else np.asarray(fmean, dtype=np.float64)
    fstd = np.ones(FEATURE_DIM) if fstd is None else np.asarray(fstd, dtype=np.float64)
    axes = AXES_BY_OP[spec.op_type]
    ext = axis_extents(spec)
    na, nl = len(axes), 2 * len(axes)
    if len(space.knobs) > MAX_KNOBS:
        raise DomainError("knob space has too many knobs for the device encoder")
    if layout.num_nodes > _lib.KT_MAX_NODES:
        raise DomainError("layout has too many nodes for the device encoder")
    if space.size >= 2**63:
        raise DomainError("knob space too large")
    t = _lib.SpecTable()
    t.n_knobs, t.n_axes, t.n_loops, t.n_nodes = len(space.knobs), na, nl, layout.num_nodes
    t.n_pairs = (layout.num_nodes - 1) // 2
    t.space_size = space.size
    names = [k.name for k in space.knobs]
    for j, k in enumerate(space.knobs):
        if len(k.values) > _lib.KT_MAX_CARD:
            raise DomainError(f"knob {k.name} has more than {_lib.KT_MAX_CARD} values")
        t.card[j] = len(k.values)
        t.card_magic[j] = (2**64 // len(k.values) + 1) if len(k.values) >= 2 else 0
    t.auto_knob = names.index("auto_unroll_max_step") if "auto_unroll_max_step" in names else -1
    t.expl_knob = names.index("unroll_explicit") if "unroll_explicit" in names else -1
    if t.auto_knob >= 0:
        for c, v in enumerate(space.knobs[t.auto_knob].values):
            t.auto_vals[c] = int(v)
    if t.expl_knob >= 0:
        for c, v in enumerate(space.knobs[t.expl_knob].values):
            t.expl_vals[c] = int(v)
    rows = [int(r) for r in layout.iterval_rows]
    if len(rows) != nl:
        raise DomainError("layout does not match the spec's loop count")
    for k, r in enumerate(rows):
        t.loop_row[k] = r
    for s in range(FEATURE_DIM):
        t.fmean[s], t.fstd[s] = float(fmean[s]), float(fstd[s])
    for a, axis in enumerate(axes):
        e = ext[axis]
        kname = f"tile_{axis}"
        t.axis_knob[a] = names.index(kname) if kname in names else -1
        t.axis_reduce[a] = 1 if axis in REDUCTION_AXES else 0
        tiles = space.knobs[t.axis_knob[a]].values if t.axis_knob[a] >= 0 else (1,)
        clamped = np.clip(np.asarray(tiles, dtype=np.int64), 1, e)
        outer = -(-e // clamped)
        lg_out = np.log2(np.maximum(outer.astype(np.float64), 1.0))
        lg_in = np.log2(np.maximum(clamped.astype(np.float64), 1.0))
        for c in range(len(tiles)):
            t.outer[a][c], t.inner[a][c] = int(outer[c]), int(clamped[c])
            t.raw_log2[0][a][c], t.raw_log2[1][a][c] = float(lg_out[c]), float(lg_in[c])
            ko, ki = a, na + a  # outer / inner loop positions
            t.nrm_ext[ko][c] = _norm32(outer[c], fmean, fstd, 0)
            t.nrm_ext[ki][c] = _norm32(clamped[c], fmean, fstd, 0)
            t.nrm_log2ext[ko][c] = _norm32(lg_out[c], fmean, fstd, 1)
            t.nrm_log2ext[ki][c] = _norm32(lg_in[c], fmean, fstd, 1)
            t.nrm_stride[ko][c] = _norm32(clamped[c], fmean, fstd, 5)
        for k, level in ((a, 0), (na + a, 1)):
            consts = {2: float(level), 3: float(t.axis_reduce[a]), 4: 0.0, 5: 1.0,
                      10: float(k + 1), 11: float(k) / max(nl - 1, 1)}
            for s, v in consts.items():
                t.nrm_const[k][s] = _norm32(v, fmean, fstd, s)
            t.nrm_unroll1[k] = _norm32(1.0, fmean, fstd, 4)
    # the scorer's per-row digit extraction (host-computed so the kernel prologue has no
    # 64-bit divisions): digit d of index v is (v // mult) % card
    cards = [len(k.values) for k in space.knobs]
    magic = lambda x: (2**64 // x + 1) if x >= 2 else 0
    for d in range(8):
        kn = (t.axis_knob[d] if d < na else -1) if d < 6 else (t.auto_knob if d == 6 else t.expl_knob)
        mult = int(np.prod(cards[kn + 1:], dtype=np.int64)) if kn >= 0 else 1
        card = cards[kn] if kn >= 0 else 1
        if mult >= 2**32:
            mult = 2**32 - 1  # (spaces >= 2^32 never reach the u32 digit path)
        t.digit_mult[d], t.digit_card[d] = mult, card
        t.digit_mult_magic[d], t.digit_card_magic[d] = magic(mult), magic(card)
    off = 0
    for a in range(6):
        t.choice_off[a] = off
        if a < na:
            off += cards[t.axis_knob[a]] if t.axis_knob[a] >= 0 else 1
    t.choice_off[6] = off
    return t


_TABLE_CACHE: dict = {}


def device_spec_table(spec, space, layout, fmean=None, fstd=None, device=None):
    """Uploaded kt_spec_table (uint8 device tensor), cached per content."""
    import ctypes

    import torch

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    key = (spec, tuple(k.values for k in space.knobs), layout.num_nodes,
           tuple(int(r) for r in layout.iterval_rows),
           None if fmean is None else np.asarray(fmean, dtype=np.float64).tobytes(),
           None if fstd is None else np.asarray(fstd, dtype=np.float64).tobytes(), str(dev))
    hit = _TABLE_CACHE.get(key)
    if hit is not None:
        return hit
    t = build_spec_table(spec, space, layout, fmean, fstd)
    raw = np.frombuffer(ctypes.string_at(ctypes.addressof(t), ctypes.sizeof(t)), dtype=np.uint8)
    buf = torch.from_numpy(raw.copy()).to(dev)
    if len(_TABLE_CACHE) > 256:
        _TABLE_CACHE.clear()
    _TABLE_CACHE[key] = buf
    return buf


_KEY_OF = operator.attrgetter("_kt_key")


def configs_to_indices(space: KnobSpace, configs) -> np.ndarray:
    """Vectorised config_index over list[KnobConfig] (validated on the host).

    Fast path: configs made by index_config (sample_configs, draw_unvisited picks, the SA /
    BO proposers) carry their index keyed to the cardinalities (kernels.KnobConfig), so a
    list converts with one pass over int attributes; anything else is re-encoded."""
    n = len(configs)
    cards_t = space.cardinalities
    if n and space.size < (1 << KEY_SHIFT):
        try:
            keys = np.fromiter(map(_KEY_OF, configs), dtype=np.int64, count=n)
        except AttributeError:
            keys = None
        if keys is not None and ((keys >> KEY_SHIFT) == card_code(cards_t)).all():
            return keys & ((1 << KEY_SHIFT) - 1)
    cards = np.array(cards_t, dtype=np.int64)
    ch = np.array([c.choices for c in configs], dtype=np.int64).reshape(len(configs), -1)
    if ch.shape[1] != len(cards):
        raise DomainError(f"config has {ch.shape[1]} choices, space has {len(cards)} knobs")
    if (ch < 0).any() or (ch >= cards).any():
        raise DomainError("choice out of range for its knob")
    mult = np.ones(len(cards), dtype=np.int64)
    for j in range(len(cards) - 2, -1, -1):
        mult[j] = mult[j + 1] * cards[j + 1]
    return ch @ mult


def encode_batch(spec: KernelSpec, space: KnobSpace, configs, layout: BatchLayout, *, device=None):
    """encode_batch (graphs.py:305-351) on the GPU: raw fp64 features (B, N, 12).

    `configs` is a list of KnobConfig (as in the reference) or an int64 tensor /
    array of config indices.  Returns a device tensor.
    """
    import torch

    from . import _lib

    tab = device_spec_table(spec, space, layout, device=device)
    dev = tab.device
    if isinstance(configs, torch.Tensor):
        idx = configs.to(dev, torch.int64)
    elif isinstance(configs, np.ndarray):
        idx = torch.from_numpy(configs.astype(np.int64)).to(dev)
    else:
        if len(configs) == 0:
            raise DomainError("empty batch")
        idx = torch.from_numpy(configs_to_indices(space, configs)).to(dev)
    b = idx.numel()
    if b == 0:
        raise DomainError("empty batch")
    out = torch.empty((b, layout.num_nodes, FEATURE_DIM), dtype=torch.float64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = _lib.load()
    with torch.cuda.device(dev):
        _lib.check(lib.kt_encode_raw(_lib.ptr(tab), _lib.ptr(idx), b, _lib.ptr(out), _lib.ptr(err),
                                     _lib.stream_handle()), "encode_batch")
    if int(err.item()):
        raise DomainError("config index out of range for the knob space")
    return out
