"""Device parity of the streaming aggregation kernels (kt_gcn_layer, kt_readout).

The layer-by-layer path equals the reference's gcn_forward / aggregate
(model.py:127-141) and embed_batch (model.py:185-194) on the same inputs:
H and u within rel 1e-4 (fp32 against fp64), and the streaming embed equals
the fused per-graph kernel (kt_embed_csr) to fp32 rounding.
"""

import numpy as np
import pytest
import torch

from oracle import kt_oracle as ko
from paper_2102_04199_b200 import graphs as pg
from paper_2102_04199_b200 import kernels as pk
from paper_2102_04199_b200 import model as pm
from paper_2102_04199_b200.errors import DomainError
from paper_2102_04199_b200.util import rng_from
from tests._shared import corpus_graphs, device_model, oracle_params, spec_of

pytestmark = pytest.mark.gpu
TEMPLATE = pg.build_super_template(pk.OP_TYPES)


def _close(dev, ref, rtol=1e-4):
    got = dev.double().cpu().numpy() if isinstance(dev, torch.Tensor) else dev
    scale = max(np.abs(ref).max(), 1e-30)
    np.testing.assert_allclose(got, ref, rtol=rtol, atol=rtol * scale)
    assert np.linalg.norm(got - ref) <= rtol * max(np.linalg.norm(ref), 1e-30)


def _feats(g_encode, g_model, rep, op="conv2d", idx=None):
    spec = spec_of(g_encode, op)
    space = pk.build_knob_space(spec)
    lay = pg.batch_layout(spec, TEMPLATE if rep == "super" else None)
    idx = g_model["score/idx"] if idx is None else idx
    return pg.encode_batch(spec, space, idx, lay), lay


@pytest.mark.parametrize("rep", ["raw", "super"])
def test_gcn_forward_batch_matches_reference(cuda_device, g_encode, g_model, rep):
    m = device_model(g_model)
    p = oracle_params(g_model)
    feats, lay = _feats(g_encode, g_model, rep)
    h = pm.gcn_forward_batch(m, feats, lay.feature_mask, lay.adjacency)
    href = ko.gcn_forward_batch(p, feats.cpu().numpy(), lay.feature_mask, lay.adjacency)
    assert h.shape == href.shape
    _close(h, href)


@pytest.mark.parametrize("rep", ["raw", "super"])
def test_streaming_embed_matches_reference_and_fused(cuda_device, g_encode, g_model, rep):
    m = device_model(g_model)
    feats, lay = _feats(g_encode, g_model, rep)
    u = pm.embed_batch_streaming(m, feats, lay.feature_mask, lay.adjacency)
    _close(u, g_model[f"score/{rep}/u"])
    fused = pm.embed_batch(m, feats, lay.feature_mask, lay.adjacency)
    np.testing.assert_allclose(u.cpu().numpy(), fused.cpu().numpy(), rtol=2e-5, atol=1e-6)


def test_aggregate_batch_matches_reference(cuda_device, g_model):
    m = device_model(g_model)
    rng = np.random.default_rng(7)
    for n in (1, 7, 25, 64):
        h = np.maximum(rng.normal(size=(333, n, 32)), 0.0).astype(np.float32)
        u = pm.aggregate_batch(torch.from_numpy(h).cuda(), m.agg)
        ref = ko.aggregate_batch(h.astype(np.float64), m.agg.sum_weights.double().cpu().numpy())
        _close(u, ref, rtol=1e-5)


def test_aggregate_batch_generic_width(cuda_device):
    """Widths that are not a power-of-two multiple of 4 take the scalar lane path."""
    rng = np.random.default_rng(3)
    for d in (5, 12, 48):
        h = rng.normal(size=(50, 9, d)).astype(np.float32)
        w = rng.normal(size=d).astype(np.float32)
        u = pm.aggregate_batch(torch.from_numpy(h).cuda(), pm.AggParams(torch.from_numpy(w).cuda()))
        _close(u, ko.aggregate_batch(h.astype(np.float64), w.astype(np.float64)), rtol=1e-5)


def test_gcn_forward_graphs_mixed_sizes(cuda_device, g_model, g_meta):
    """Raw graphs of 17 / 21 / 25 nodes (three adjacency patterns) in one segmented batch."""
    m = device_model(g_model)
    p = oracle_params(g_model)
    graphs = corpus_graphs(g_meta, super_graph=False)[::3]
    cg = []
    for x, adj, mask in graphs:
        n = x.shape[0]
        nodes = [pg.GraphNode("root")] + [
            pg.GraphNode("iterval" if i % 2 == 0 else "for_node", feature=x[i] if mask[i] else None)
            for i in range(1, n)]
        edges = [(0, 2 * i + 1) for i in range((n - 1) // 2)] + [(2 * i + 1, 2 * i + 2) for i in range((n - 1) // 2)]
        cg.append(pg.CodeGraph(nodes=nodes, edges=edges))
    assert sorted({x.shape[0] for x, _, _ in graphs}) == [17, 21, 25]
    h, node_ptr = pm.gcn_forward_graphs(m, cg)
    npt = node_ptr.cpu().numpy()
    for g, (x, adj, mask) in enumerate(graphs):
        href = ko.gcn_forward_batch(p, x[None], mask, adj)[0]
        _close(h[npt[g]:npt[g + 1]], href)
    u = pm.aggregate_batch(h, m.agg, node_ptr)
    uref = np.stack([ko.embed_batch(p, x[None], mask, adj)[0] for x, adj, mask in graphs])
    _close(u, uref)


def test_gcn_layer_generic_dims(cuda_device, g_encode, g_model):
    """Odd layer widths (no bulk copies, scalar transform) against the oracle."""
    m = pm.init_model(rng_from("agg-odd"), gcn_dims=(5, 7), head_hidden=(6,), device="cuda")
    p = {"gcn": [w.double().cpu().numpy() for w in m.gcn.layers], "fmean": m.feature_norm.mean,
         "fstd": m.feature_norm.std}
    feats, lay = _feats(g_encode, g_model, "super")
    h = pm.gcn_forward_batch(m, feats, lay.feature_mask, lay.adjacency)
    _close(h, ko.gcn_forward_batch(p, feats.cpu().numpy(), lay.feature_mask, lay.adjacency))


def test_gcn_layer_large_batch_position_invariant(cuda_device, g_encode, g_model):
    """200k graphs through the bulk-copy pipeline: every tile position gives the same rows."""
    m = device_model(g_model)
    spec = spec_of(g_encode, "conv2d")
    space = pk.build_knob_space(spec)
    lay = pg.batch_layout(spec, TEMPLATE)
    idx = rng_from("agg-large").integers(0, space.size, 200_003)
    feats = pg.encode_batch(spec, space, idx, lay)
    h = pm.gcn_forward_batch(m, feats, lay.feature_mask, lay.adjacency)
    pick = np.array([0, 1, 7, 8, 9, 1000, 99_999, 200_002])
    h_small = pm.gcn_forward_batch(m, feats[pick], lay.feature_mask, lay.adjacency)
    assert torch.equal(h[pick], h_small)
    p = oracle_params(g_model)
    _close(h[pick], ko.gcn_forward_batch(p, feats[pick].cpu().numpy(), lay.feature_mask, lay.adjacency))
    u = pm.aggregate_batch(h, m.agg)
    assert torch.equal(u[pick], pm.aggregate_batch(h_small, m.agg))


def test_streaming_errors(cuda_device, g_model):
    m = device_model(g_model)
    with pytest.raises(DomainError):
        pm.gcn_forward_batch(m, np.zeros((0, 25, 12)), np.ones(25, bool), np.eye(25))
    with pytest.raises(DomainError):
        pm.gcn_forward_batch(m, np.zeros((3, 25, 11)), np.ones(25, bool), np.eye(25))
    with pytest.raises(DomainError):
        pm.aggregate_batch(torch.zeros((2, 3, 31), device="cuda"), m.agg)


@pytest.mark.parametrize("variant", ["KT_AGG_NOTM", "KT_AGG_FFMA"])
def test_layer_kernel_variants_agree(cuda_device, g_encode, g_model, monkeypatch, variant):
    """Every layer kernel gives the same H (fp32-level) on 50k super graphs: the default
    TMA-pipelined path (swizzled tensor maps for uniform graphs) against the 1-D bulk
    pipeline (NOTM), the unpipelined tensor-core kernel (TC1) and the FFMA2 warp kernel."""
    m = device_model(g_model)
    spec = spec_of(g_encode, "conv2d")
    space = pk.build_knob_space(spec)
    lay = pg.batch_layout(spec, TEMPLATE)
    feats = pg.encode_batch(spec, space, rng_from("agg-var").integers(0, space.size, 50_001), lay)
    h_def = pm.gcn_forward_batch(m, feats, lay.feature_mask, lay.adjacency)
    monkeypatch.setenv(variant, "1")
    h_var = pm.gcn_forward_batch(m, feats, lay.feature_mask, lay.adjacency)
    monkeypatch.delenv(variant)
    _close(h_def, h_var.double().cpu().numpy(), rtol=2e-5)
