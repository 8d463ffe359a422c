"""Index-based training datasets, materialised on the device.

The reference keeps its training corpus index-based -- per kernel class a
KernelRecords of config indices, measured GFLOPS and feasibility
(harness.py:97-114), persisted by save_dataset / load_dataset as kernels.yaml +
samples.csv + manifest.json (harness.py:195-252) -- and rebuilds a CodeGraph per
sample in dataset_samples (harness.py:179-192) before any training can start
(3.7 s for the 9,400-sample corpus).  Here each class's index vector goes
through the device encoder (kt_encode_raw, graphs.py:305-351) in one launch, and
the packed segmented-CSR batch the training kernels read (model.PackedGraphs) is
assembled with array arithmetic: per class one layout (batch_layout,
graphs.py:278-302) tiled over its samples.  No CodeGraph is built unless a
caller asks a sample for `.graph`.

IndexedDataset behaves as the reference's list of LabeledSample wherever the
package takes one (dataset_norms, pretrain, sample_meta_tasks, MetaTrainer,
grad via grad_indexed): those take the packed batch directly.
"""

from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from .errors import ConfigError, DomainError
from .graphs import batch_layout, build_super_template, config_graph, encode_batch
from .kernels import OP_TYPES, KernelSpec, KnobSpace, build_knob_space, index_config
from .model import LABEL_FLOOR_GFLOPS, PackedGraphs
from .util import stable_digest

_SPEC_FIELDS = ("op_type", "input_size", "in_channels", "out_channels", "kernel_size", "stride", "padding")


@dataclass
class KernelRecords:
    """harness.py:97-102: one kernel class's measured configs."""
    spec: KernelSpec
    indices: np.ndarray   # int64 config indices into build_knob_space(spec)
    gflops: np.ndarray    # float64
    feasible: np.ndarray  # bool


def _as_spec(s) -> KernelSpec:
    if isinstance(s, KernelSpec):
        return s
    return KernelSpec(*(getattr(s, f) for f in _SPEC_FIELDS))


def _spec_signature(spec: KernelSpec) -> str:
    # kernels.py:67-72 (padding is not part of the class identity)
    return (f"{spec.op_type}/{spec.input_size}/{spec.in_channels}/{spec.out_channels}/"
            f"{spec.kernel_size}/{spec.stride}")


def content_hash(params: dict, entries: list) -> str:
    """Dataset.content_hash (harness.py:112-119)."""
    parts = [json.dumps(params, sort_keys=True)]
    for e in entries:
        parts += [_spec_signature(e.spec), np.asarray(e.indices, dtype=np.int64).tobytes(),
                  np.asarray(e.gflops, dtype=np.float64).tobytes(), np.asarray(e.feasible, dtype=bool).tobytes()]
    return stable_digest("dataset", tuple(parts))


def load_records(in_dir: str, verify: bool = True) -> tuple:
    """load_dataset (harness.py:219-252): (params dict, [KernelRecords]); the manifest's
    content hash is checked as the reference does (ConfigError on mismatch)."""
    import yaml

    mpath = os.path.join(in_dir, "manifest.json")
    if not os.path.exists(mpath):
        raise ConfigError(f"no dataset manifest at {mpath}")
    with open(mpath, encoding="utf-8") as f:
        manifest = json.load(f)
    with open(os.path.join(in_dir, "kernels.yaml"), encoding="utf-8") as f:
        kdata = yaml.safe_load(f.read())
    if not isinstance(kdata, list):
        raise ConfigError("kernel file must be a list of specs")
    try:
        specs = [KernelSpec(str(d["op_type"]), int(d["input_size"]), int(d["in_channels"]), int(d["out_channels"]),
                            int(d["kernel_size"]), int(d.get("stride", 3)), int(d.get("padding", 1))) for d in kdata]
    except KeyError as e:
        raise ConfigError(f"kernel spec missing field {e.args[0]!r}") from e
    buckets = {i: ([], [], []) for i in range(len(specs))}
    with open(os.path.join(in_dir, "samples.csv"), encoding="utf-8") as f:
        lines = f.read().splitlines()
    for line in lines[1:]:
        if not line.strip():
            continue
        ki, idx, g, fe = line.split(",")
        b = buckets[int(ki)]
        b[0].append(int(idx))
        b[1].append(float(g))
        b[2].append(bool(int(fe)))
    entries = [KernelRecords(spec, np.array(b[0], dtype=np.int64), np.array(b[1], dtype=np.float64),
                             np.array(b[2], dtype=bool)) for spec, b in ((specs[i], buckets[i]) for i in buckets)]
    if verify and content_hash(manifest["params"], entries) != manifest["content_hash"]:
        raise ConfigError(f"dataset at {in_dir} does not match its manifest hash")
    return manifest["params"], entries


class IndexedSample:
    """A LabeledSample (meta.py:37-45) that knows its config index instead of holding a
    graph; `.graph` builds the CodeGraph on demand for reference-API callers."""

    __slots__ = ("spec", "space", "index", "kernel_class", "label_gflops", "position", "_template", "_graph")

    def __init__(self, spec, space, index, kernel_class, label_gflops, position, template):
        self.spec, self.space, self.index = spec, space, index
        self.kernel_class, self.label_gflops, self.position = kernel_class, label_gflops, position
        self._template, self._graph = template, None

    @property
    def graph(self):
        if self._graph is None:
            self._graph = config_graph(self.spec, index_config(self.space, self.index), self.space, self._template)
        return self._graph

    def __repr__(self):
        return f"IndexedSample({self.kernel_class!r}, idx={self.index}, gflops={self.label_gflops!r})"


class IndexedDataset:
    """dataset_samples (harness.py:179-192) as one device-resident packed batch.

    Sample order, labels (max(gflops, LABEL_FLOOR_GFLOPS), infeasible -> floor) and
    kernel classes (spec signature) are the reference's; the packed tensors equal
    model.pack_graphs over the materialised graphs (features to the encoder's 1 ulp
    on the two log2 slots, everything else bit-exact)."""

    def __init__(self, entries: list, augmented: bool, *, device=None):
        if not entries:
            raise DomainError("empty dataset")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        template = build_super_template(OP_TYPES) if augmented else None
        self.augmented = augmented
        self.entries = [KernelRecords(_as_spec(e.spec), np.asarray(e.indices, dtype=np.int64),
                                      np.asarray(e.gflops, dtype=np.float64), np.asarray(e.feasible, dtype=bool))
                        for e in entries]
        self.samples: list = []
        feats, masks, sizes, rows, cols, vals = [], [], [], [], [], []
        node_base = 0
        for e in self.entries:
            n = e.indices.size
            if n == 0:
                continue
            space: KnobSpace = build_knob_space(e.spec)
            cls = _spec_signature(e.spec)
            for i in range(n):
                self.samples.append(IndexedSample(e.spec, space, int(e.indices[i]), cls,
                                                  max(float(e.gflops[i]), LABEL_FLOOR_GFLOPS), len(self.samples),
                                                  template))
            lay = batch_layout(e.spec, template)
            nn = lay.num_nodes
            x = encode_batch(e.spec, space, e.indices, lay, device=dev)  # (n, nn, 12) fp64, one launch
            feats.append(x.reshape(n * nn, x.shape[2]))
            masks.append(np.tile(lay.feature_mask.astype(np.uint8), n))
            sizes.append(np.full(n, nn, dtype=np.int64))
            r, c = np.nonzero(lay.adjacency)  # row-major, as pack_graphs / graph_to_tensors
            offs = node_base + nn * np.arange(n, dtype=np.int64)[:, None]
            rows.append((r[None, :] + offs).ravel())
            cols.append((c[None, :] + offs).ravel())
            vals.append(np.tile(lay.adjacency[r, c], n))
            node_base += n * nn
        if not self.samples:
            raise DomainError("empty dataset")
        sizes = np.concatenate(sizes)
        node_ptr = np.concatenate([[0], np.cumsum(sizes)])
        rows = np.concatenate(rows)
        row_ptr = np.zeros(node_ptr[-1] + 1, dtype=np.int64)
        np.add.at(row_ptr, rows + 1, 1)
        row_ptr = np.cumsum(row_ptr)
        up = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)
        self.packed = PackedGraphs(torch.cat(feats).contiguous(), up(np.concatenate(masks), np.uint8),
                                   up(node_ptr, np.int64), up(row_ptr, np.int32), up(np.concatenate(cols), np.int32),
                                   up(np.concatenate(vals), np.float32), int(sizes.max()), len(self.samples))
        self.labels = np.array([s.label_gflops for s in self.samples], dtype=np.float64)
        self.device = dev

    @classmethod
    def load(cls, in_dir: str, augmented: bool, *, device=None, verify: bool = True) -> "IndexedDataset":
        """load_dataset (harness.py:219) + dataset_samples (harness.py:179) in one step."""
        return cls(load_records(in_dir, verify)[1], augmented, device=device)

    @classmethod
    def from_reference(cls, ds, augmented: bool, *, device=None) -> "IndexedDataset":
        """From a reference Dataset object (harness.py:105-110): its .entries records."""
        return cls(list(ds.entries), augmented, device=device)

    # list-of-LabeledSample protocol
    def __len__(self):
        return len(self.samples)

    def __iter__(self):
        return iter(self.samples)

    def __getitem__(self, i):
        return self.samples[i]

    def feature_rows(self) -> np.ndarray:
        """The iterval rows of every sample, stacked in sample order (host fp64)."""
        x = self.packed.feats.cpu().numpy()
        return x[self.packed.mask.cpu().numpy().astype(bool)]

    def norms(self) -> tuple:
        """dataset_norms (meta.py:81-101) from the device-encoded features."""
        from .model import FeatureNorm, LabelNorm

        stacked = self.feature_rows()
        std = stacked.std(axis=0)
        labels = [math.log2(max(v, LABEL_FLOOR_GFLOPS)) for v in self.labels]
        lstd = float(np.std(labels))
        return (FeatureNorm(stacked.mean(axis=0), np.where(std < 1e-12, 1.0, std)),
                LabelNorm(float(np.mean(labels)), lstd if lstd >= 1e-12 else 1.0))


def packed_of(dataset, dev) -> PackedGraphs:
    """The packed batch of a dataset: IndexedDataset's own, else pack_graphs of the graphs."""
    from .model import pack_graphs

    if isinstance(dataset, IndexedDataset):
        if dataset.device != torch.device(dev):
            raise DomainError("dataset lives on another device than the model")
        return dataset.packed
    return pack_graphs([s.graph for s in dataset], dev)


def grad_indexed(m, ds: IndexedDataset, sample_idx, scope: str = "all"):
    """grad(m, [(ds[i].graph, ds[i].label) for i in sample_idx], scope) (model.py:218-285)
    without materialising graphs: the kernel gathers the batch from the resident
    dataset by position (SURVEY.md 8(b) `grad_indexed`)."""
    from .model import _grad_packed, flat_params, grads_from_flat, normalize_label

    pick = np.asarray(sample_idx, dtype=np.int64).ravel()
    if pick.size == 0:
        raise DomainError("empty batch")
    if pick.min() < 0 or pick.max() >= len(ds):
        raise DomainError("sample index out of range")
    dev = flat_params(m).device
    ys = np.array([normalize_label(m, float(ds.labels[i])) for i in pick], dtype=np.float32)
    gi = torch.from_numpy(pick).to(dev)
    loss, g, _ = _grad_packed(m, packed_of(ds, dev), torch.from_numpy(ys).to(dev), scope, gi)
    return float(loss.item()), grads_from_flat(g, m)
