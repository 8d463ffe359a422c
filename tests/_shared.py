"""Helpers shared by the CPU and GPU parity tests (fixture decoding)."""

from __future__ import annotations

import numpy as np

from oracle import kt_oracle as ko
from paper_2102_04199_b200.kernels import OP_TYPES, KernelSpec

GOLDEN_SPEC_FIELDS = ("input_size", "in_channels", "out_channels", "kernel_size", "stride", "padding")


def spec_of(g, op) -> KernelSpec:
    vals = [int(v) for v in g[f"{op}/spec"]]
    return KernelSpec(op, *vals)


def oracle_params(g_model) -> dict:
    p = {k[2:]: v for k, v in g_model.items() if k.startswith("p/")}
    n_gcn = sum(1 for k in p if k.startswith("gcn"))
    n_head = sum(1 for k in p if k.startswith("hw"))
    return {
        "gcn": [p[f"gcn{i}"] for i in range(n_gcn)],
        "agg": p["agg"],
        "head_w": [p[f"hw{i}"] for i in range(n_head)],
        "head_b": [p[f"hb{i}"] for i in range(n_head)],
        "fmean": p["fmean"],
        "fstd": p["fstd"],
        "lmean": float(p["lnorm"][0]),
        "lstd": float(p["lnorm"][1]),
    }


def head_shapes(params) -> list:
    return [w.shape for w in params["head_w"]]


def corpus_graphs(g_meta, super_graph=True):
    """Rebuild the golden corpus (ops x configs) as oracle (X raw, adj, mask) triples."""
    from tests.conftest import load_golden

    enc = load_golden("encode")
    out = []
    cache = {}
    for op_i, idx in zip(g_meta["op"], g_meta["idx"]):
        op = OP_TYPES[int(op_i)]
        if op not in cache:
            s = spec_of(enc, op)
            ext = ko.extents(op, s.input_size, s.in_channels, s.out_channels, s.kernel_size,
                             s.stride, s.padding)
            knobs = ko.knob_lists(op, ext)
            adj, rows, mask = ko.layout(op, super_graph)
            cache[op] = (ext, knobs, adj, rows, mask)
        ext, knobs, adj, rows, mask = cache[op]
        ch = ko.decode([len(v) for _, v in knobs], np.array([idx]))
        x = ko.encode(op, ext, knobs, ch, adj.shape[0], rows)[0]
        out.append((x, adj, mask))
    return out


class _NS:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def device_model(g_model, device=None):
    """Product ModelState (fp32, device) holding the golden fp64 parameters."""
    from paper_2102_04199_b200.model import from_reference

    p = oracle_params(g_model)
    ref = _NS(
        gcn=_NS(layers=p["gcn"]), agg=_NS(sum_weights=p["agg"]),
        head=_NS(weights=p["head_w"], biases=p["head_b"]),
        feature_norm=_NS(mean=p["fmean"], std=p["fstd"]),
        label_norm=_NS(mean=p["lmean"], std=p["lstd"]),
    )
    return from_reference(ref, device=device)


from tests.parity_tools import expand_unique, rank_parity, sweep_indices  # noqa: E402,F401
