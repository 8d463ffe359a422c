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


def expand_unique(g, key):
    """Undo make_goldens.unique_rows: rows = uniq[inv]."""
    return g[f"{key}_uniq"][g[f"{key}_inv"]]


def sweep_indices(n, size):
    """The C5 fixture's candidates: n distinct indices from rng_from("sweep", 0), first
    occurrences kept (make_goldens.sweep_indices)."""
    from paper_2102_04199_b200.util import rng_from

    rng = rng_from("sweep", 0)
    out, seen = [], set()
    while len(out) < n:
        for v in rng.integers(0, size, n - len(out)):
            if int(v) not in seen:
                seen.add(int(v))
                out.append(int(v))
    return np.array(out, dtype=np.int64)


def rank_parity(got, ref_top, idx, z_ref, tol=1e-5) -> dict:
    """Ranking parity after tie-class canonicalisation.

    `got`: the device's top-k indices in order; `ref_top`: the reference's rank_history
    top-k over its fp64 scores; `idx`, `z_ref`: every candidate and its reference score.
    Both orders are total orders on (-score, index), so an exact-tie class (identical
    encoded features => bitwise-equal reference scores) is ordered by index in both, and
    any disagreement is a pair of candidates the two orders place differently.  Every
    such pair among the union of both lists is counted: a *tie flip* when the reference
    scores are equal (an exact-tie class left index order: a failure), a *near-tie flip*
    when they differ by at most tol * |z| (reported), a *hard flip* otherwise (a failure).
    """
    got = [int(v) for v in got]
    ref_top = [int(v) for v in ref_top]
    zmap = dict(zip(np.asarray(idx).tolist(), np.asarray(z_ref, dtype=np.float64).tolist()))
    union = list(dict.fromkeys(got + ref_top))
    k = len(got)
    gpos = {v: p for p, v in enumerate(got)}
    u = np.array(union, dtype=np.int64)
    z = np.array([zmap[v] for v in union])
    gp = np.array([gpos.get(v, k) for v in union])
    # reference order: a before b iff (-z_a, a) < (-z_b, b)
    ref_before = (z[:, None] > z[None, :]) | ((z[:, None] == z[None, :]) & (u[:, None] < u[None, :]))
    gpu_before = gp[:, None] < gp[None, :]
    both_out = (gp[:, None] == k) & (gp[None, :] == k)
    flip = gpu_before & ~ref_before & ~both_out
    np.fill_diagonal(flip, False)
    gap = np.abs(z[:, None] - z[None, :])
    near = gap <= tol * np.maximum(np.abs(z[:, None]), np.abs(z[None, :]))
    tie = gap == 0.0
    return {"exact": got == ref_top, "hard_flips": int((flip & ~near).sum()),
            "tie_flips": int((flip & tie).sum()), "near_flips": int((flip & near & ~tie).sum()),
            "max_flip_gap": float(gap[flip].max()) if flip.any() else 0.0}
