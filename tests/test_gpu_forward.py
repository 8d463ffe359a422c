"""Device parity of the forward path (encoder, fused scorer, general embed, head, top-k).

Runs on a B200 (`-m gpu`).  Every call goes through libkerntune_b200.so.
Tolerances: encoder bit-exact (fp64), except log2 slots 7/9 which may differ
by one fp64 ulp (CUDA log2 vs numpy); predicted GFLOPS within rel 1e-4 (the
north-star bar), i.e. |dz| <= 1e-4 / (ln2 * sigma_y); embeddings rel 1e-4.
"""

import math

import numpy as np
import pytest
import torch

from oracle import kt_oracle as ko
from paper_2102_04199_b200 import graphs as pg
from paper_2102_04199_b200 import kernels as pk
from paper_2102_04199_b200 import model as pm
from paper_2102_04199_b200 import search as ps
from paper_2102_04199_b200.util import rng_from
from tests._shared import corpus_graphs, device_model, oracle_params, spec_of

pytestmark = pytest.mark.gpu
OPS = pk.OP_TYPES
TEMPLATE = pg.build_super_template(OPS)


def _layout(spec, rep):
    return pg.batch_layout(spec, TEMPLATE if rep == "super" else None)


def _assert_gflops_close(z_dev, z_ref, lstd, rtol=1e-4):
    z = z_dev.double().cpu().numpy()
    # GFLOPS = 2^(z*sigma + mu): rel error = 2^(dz*sigma) - 1
    rel = np.abs(np.exp2((z - z_ref) * lstd) - 1.0)
    assert rel.max() < rtol, f"max rel GFLOPS error {rel.max():.3e}"


@pytest.mark.parametrize("rep", ["raw", "super"])
@pytest.mark.parametrize("op", OPS)
def test_encode_batch_device_matches_reference(cuda_device, g_encode, op, rep):
    spec = spec_of(g_encode, op)
    space = pk.build_knob_space(spec)
    lay = _layout(spec, rep)
    x = pg.encode_batch(spec, space, g_encode[f"{op}/idx"], lay).cpu().numpy()
    ref = g_encode[f"{op}/{rep}/feats"]
    rows = lay.iterval_rows
    got = x[:, rows, :]
    assert not np.delete(x, rows, axis=1).any()
    exact = [s for s in range(12) if s not in (7, 9)]
    assert got[..., exact].tobytes() == ref[..., exact].tobytes()
    ulp = np.abs(got[..., [7, 9]].view(np.int64) - ref[..., [7, 9]].view(np.int64))
    assert ulp.max() <= 1


def test_encode_batch_from_knob_configs(cuda_device, g_encode):
    spec = spec_of(g_encode, "depthwise")
    space = pk.build_knob_space(spec)
    cfgs = [pk.KnobConfig(tuple(int(v) for v in c)) for c in g_encode["depthwise/choices"]]
    lay = _layout(spec, "super")
    a = pg.encode_batch(spec, space, cfgs, lay)
    b = pg.encode_batch(spec, space, g_encode["depthwise/idx"], lay)
    assert torch.equal(a, b)


def test_encode_rejects_out_of_range(cuda_device, g_encode):
    spec = spec_of(g_encode, "conv2d")
    space = pk.build_knob_space(spec)
    with pytest.raises(pg.DomainError):
        pg.encode_batch(spec, space, np.array([space.size]), _layout(spec, "super"))


ENGINES = ["tc", "fp32"]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("rep", ["raw", "super"])
def test_fused_scorer_matches_reference(cuda_device, g_encode, g_model, rep, engine):
    m = device_model(g_model)
    spec = spec_of(g_encode, "conv2d")
    space = pk.build_knob_space(spec)
    z, u = ps.score_indices(m, spec, space, _layout(spec, rep), g_model["score/idx"], want_u=True, engine=engine)
    _assert_gflops_close(z, g_model[f"score/{rep}/z"], m.label_norm.std)
    np.testing.assert_allclose(u.double().cpu().numpy(), g_model[f"score/{rep}/u"], rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("op", OPS)
def test_fused_scorer_all_ops_vs_oracle(cuda_device, g_encode, g_model, op, engine):
    p = oracle_params(g_model)
    m = device_model(g_model)
    spec = spec_of(g_encode, op)
    space = pk.build_knob_space(spec)
    s = spec
    ext = ko.extents(op, s.input_size, s.in_channels, s.out_channels, s.kernel_size, s.stride, s.padding)
    knobs = ko.knob_lists(op, ext)
    for rep in ("raw", "super"):
        adj, rows, mask = ko.layout(op, rep == "super")
        x = ko.encode(op, ext, knobs, g_encode[f"{op}/choices"], adj.shape[0], rows)
        zref = ko.score(p, x, mask, adj)
        z = ps.score_indices(m, spec, space, _layout(spec, rep), g_encode[f"{op}/idx"], engine=engine)
        _assert_gflops_close(z, zref, m.label_norm.std)


@pytest.mark.parametrize("engine", ENGINES)
def test_scorer_contiguous_range_equals_index_list(cuda_device, g_model, engine):
    m = device_model(g_model)
    spec = pk.KernelSpec("conv2d", 56, 64, 64, 3, 3, 1)
    space = pk.build_knob_space(spec)
    lay = _layout(spec, "super")
    base = 123_456_789
    a = ps.score_indices(m, spec, space, lay, base=base, count=5000, engine=engine)
    b = ps.score_indices(m, spec, space, lay, np.arange(base, base + 5000), engine=engine)
    assert torch.equal(a, b)


def test_tensor_core_and_fp32_scorers_agree(cuda_device, g_model):
    """3xTF32 tcgen05 kernel vs the independent FFMA2 kernel on 100k candidates (both vs fp64 elsewhere)."""
    m = device_model(g_model)
    spec = pk.KernelSpec("conv2d", 56, 64, 64, 3, 3, 1)
    space = pk.build_knob_space(spec)
    lay = _layout(spec, "super")
    idx = np.random.default_rng(11).integers(0, space.size, 100_000)
    a = ps.score_indices(m, spec, space, lay, idx, engine="tc").double()
    b = ps.score_indices(m, spec, space, lay, idx, engine="fp32").double()
    assert torch.isfinite(a).all()
    assert (a - b).abs().max().item() <= 2e-5 * max(1.0, b.abs().max().item())


@pytest.mark.parametrize("engine", ENGINES)
def test_scorer_is_batch_position_invariant_and_deterministic(cuda_device, g_model, engine):
    """Per-candidate arithmetic must not depend on the batch (ties stay ties)."""
    m = device_model(g_model)
    spec = pk.KernelSpec("conv2d", 56, 64, 64, 3, 3, 1)
    space = pk.build_knob_space(spec)
    lay = _layout(spec, "super")
    rng = np.random.default_rng(7)
    idx = rng.integers(0, space.size, 3001)
    z_full = ps.score_indices(m, spec, space, lay, idx, engine=engine).cpu().numpy()
    perm = rng.permutation(idx.size)
    z_perm = ps.score_indices(m, spec, space, lay, idx[perm], engine=engine).cpu().numpy()
    assert z_perm.tobytes() == z_full[perm].tobytes()
    for b in (1, 7, 64, 65, 121):
        z_small = ps.score_indices(m, spec, space, lay, idx[:b], engine=engine).cpu().numpy()
        assert z_small.tobytes() == z_full[:b].tobytes()
    assert ps.score_indices(m, spec, space, lay, idx, engine=engine).cpu().numpy().tobytes() == z_full.tobytes()


@pytest.mark.parametrize("engine", ENGINES)
def test_scorer_tie_classes_match_reference(cuda_device, g_model, engine):
    """Identical encoded features => bit-identical scores (the reference's exact ties)."""
    m = device_model(g_model)
    spec = pk.KernelSpec("conv2d", 56, 64, 64, 3, 3, 1)
    space = pk.build_knob_space(spec)
    lay = _layout(spec, "super")
    idx = np.random.default_rng(3).integers(0, space.size, 20000)
    feats = pg.encode_batch(spec, space, idx, lay).cpu().numpy()
    z = ps.score_indices(m, spec, space, lay, idx, engine=engine).cpu().numpy()
    keys = {}
    for f, v in zip(feats.reshape(len(idx), -1), z):
        keys.setdefault(f.tobytes(), set()).add(v.tobytes())
    assert all(len(s) == 1 for s in keys.values())
    assert len(keys) < len(idx)  # the space really is tie-heavy


def test_scorer_rejects_bad_index(cuda_device, g_model):
    m = device_model(g_model)
    spec = pk.KernelSpec("conv2d", 56, 64, 64, 3, 3, 1)
    space = pk.build_knob_space(spec)
    with pytest.raises(pg.DomainError):
        ps.score_indices(m, spec, space, _layout(spec, "super"), np.array([0, -1]))


@pytest.mark.parametrize("rep", ["raw", "super"])
def test_embed_batch_general_matches_reference(cuda_device, g_encode, g_model, rep):
    m = device_model(g_model)
    spec = spec_of(g_encode, "conv2d")
    space = pk.build_knob_space(spec)
    lay = _layout(spec, rep)
    feats = pg.encode_batch(spec, space, g_model["score/idx"], lay)
    u = pm.embed_batch(m, feats, lay.feature_mask, lay.adjacency)
    np.testing.assert_allclose(u.double().cpu().numpy(), g_model[f"score/{rep}/u"], rtol=1e-4, atol=1e-5)
    z = pm.head_forward_batch(u, m.head)
    _assert_gflops_close(z, g_model[f"score/{rep}/z"], m.label_norm.std)


def test_head_forward_tiled_equals_warp_kernel(cuda_device, g_model, monkeypatch):
    """kt_head_forward's tiled kernel (64-row tiles, parameters in shared memory) computes every
    output with the warp-per-row kernel's fmaf order: bit-identical, at any batch position."""
    m = device_model(g_model)
    u = torch.from_numpy(np.abs(rng_from("head-tile").normal(size=(1000, 64))).astype(np.float32)).cuda()
    z_tile = pm.head_forward_batch(u, m.head)
    pick = torch.tensor([0, 63, 64, 999], device=u.device)
    assert torch.equal(pm.head_forward_batch(u[pick].contiguous(), m.head), z_tile[pick])
    monkeypatch.setenv("KT_HEADF_WARP", "1")
    assert torch.equal(pm.head_forward_batch(u, m.head), z_tile)


def test_embed_graphs_mixed_sizes_matches_reference(cuda_device, g_encode, g_model):
    m = device_model(g_model)
    graphs = []
    for op_i, idx in zip(g_model["mixed/op"], g_model["mixed/idx"]):
        op = OPS[int(op_i)]
        spec = spec_of(g_encode, op)
        space = pk.build_knob_space(spec)
        graphs.append(pg.config_graph(spec, pk.index_config(space, int(idx)), space, template=TEMPLATE))
    u, z = pm.embed_graphs(m, graphs, with_scores=True)
    np.testing.assert_allclose(u.double().cpu().numpy(), g_model["mixed/u"], rtol=1e-4, atol=1e-5)
    _assert_gflops_close(z, g_model["mixed/z"], m.label_norm.std)
    assert math.isclose(pm.forward(graphs[3], m), float(g_model["mixed/z"][3]), rel_tol=1e-4, abs_tol=1e-5)


def test_embed_graphs_small_and_large_batch_paths_agree(cuda_device, g_encode, g_model):
    """kt_embed_csr runs one CTA per graph for B <= 148 (single-graph API) and one warp
    per graph above; both keep the per-element operation order, so bit-identical."""
    m = device_model(g_model)
    spec = spec_of(g_encode, OPS[0])
    space = pk.build_knob_space(spec)
    graphs = [pg.config_graph(spec, pk.index_config(space, int(i)), space, template=TEMPLATE)
              for i in range(0, 300 * 7, 7)]
    u_big, z_big = pm.embed_graphs(m, graphs, with_scores=True)
    u_small, z_small = pm.embed_graphs(m, graphs[:100], with_scores=True)
    assert torch.equal(u_big[:100], u_small) and torch.equal(z_big[:100], z_small)
    for i in (0, 57, 299):
        u1, z1 = pm.embed_graphs(m, [graphs[i]], with_scores=True)
        assert torch.equal(u1[0], u_big[i]) and torch.equal(z1[0], z_big[i])
        assert pm.forward(graphs[i], m) == float(z_big[i])


def test_raw_segmented_batch_vs_oracle(cuda_device, g_model, g_meta):
    """Raw graphs of 17/21/25 nodes in one segmented CSR batch."""
    m = device_model(g_model)
    p = oracle_params(g_model)
    graphs = corpus_graphs(g_meta, super_graph=False)[::5]
    cg = []
    for x, adj, mask in graphs:
        n = x.shape[0]
        nodes = [pg.GraphNode("root")] + [
            pg.GraphNode("iterval" if i % 2 == 0 else "for_node", feature=x[i] if mask[i] else None)
            for i in range(1, n)]
        edges = [(0, 2 * i + 1) for i in range((n - 1) // 2)] + [(2 * i + 1, 2 * i + 2) for i in range((n - 1) // 2)]
        cg.append(pg.CodeGraph(nodes=nodes, edges=edges))
    u, z = pm.embed_graphs(m, cg, with_scores=True)
    zref = np.array([ko.score(p, x[None], mask, adj)[0] for x, adj, mask in graphs])
    assert sorted({x.shape[0] for x, _, _ in graphs}) == [17, 21, 25]
    _assert_gflops_close(z, zref, m.label_norm.std)


def test_topk_matches_rank_history(cuda_device, g_rank):
    scores = torch.tensor(g_rank["scores"], dtype=torch.float32, device="cuda")
    idx = torch.tensor(g_rank["idx"], dtype=torch.int64, device="cuda")
    visited = set(int(v) for v in g_rank["visited"])
    ti, ts = ps.topk(scores, 128, idx, visited=visited)
    # fp32 copy of the scores: rank with the oracle on the same fp32 values
    want = ko.rank_history(g_rank["idx"], g_rank["scores"].astype(np.float32), visited, 128)
    assert ti.cpu().tolist() == want
    assert ti.cpu().tolist() == [int(v) for v in g_rank["top"]]


def test_topk_large_and_merge(cuda_device, g_model):
    m = device_model(g_model)
    spec = pk.KernelSpec("conv2d", 56, 64, 64, 3, 3, 1)
    space = pk.build_knob_space(spec)
    lay = _layout(spec, "super")
    n = 300_000
    base = 7_000_000
    z = ps.score_indices(m, spec, space, lay, base=base, count=n)
    ti, ts = ps.topk(z, 512, base=base)
    zc = z.cpu().numpy()
    order = np.lexsort((np.arange(n), -zc.astype(np.float64)))[:512]
    assert ti.cpu().numpy().tolist() == (order + base).tolist()
    assert np.array_equal(ts.cpu().numpy(), zc[order])
    # two "ranks" worth of shards merged == global
    h = n // 2
    a_i, a_s = ps.topk(z[:h], 512, base=base)
    b_i, b_s = ps.topk(z[h:], 512, base=base + h)
    mi, ms = ps.topk_merge(torch.cat([a_s, b_s]), torch.cat([a_i, b_i]), 512)
    assert torch.equal(mi, ti) and torch.equal(ms, ts)


def test_predictor_callable_contract(cuda_device, g_model):
    m = device_model(g_model)
    spec = pk.KernelSpec("conv2d", 56, 64, 64, 3, 3, 1)
    space = pk.build_knob_space(spec)
    pred = ps.CostModelPredictor(m, spec, space, template=TEMPLATE)
    cfgs = pk.sample_configs(space, 16, np.random.default_rng(0))
    e = pred(cfgs)
    assert e.dtype == np.float64 and e.shape == (16,)
    z, u = pred.meta_scores(cfgs)
    assert np.array_equal(z, e) and u.shape == (16, 64)


def test_single_graph_api(cuda_device, g_model):
    m = device_model(g_model)
    spec = pk.KernelSpec("conv2d", 56, 64, 64, 3, 3, 1)
    space = pk.build_knob_space(spec)
    g = pg.config_graph(spec, pk.index_config(space, 31337), space, template=TEMPLATE)
    lay = _layout(spec, "super")
    z = ps.score_indices(m, spec, space, lay, np.array([31337])).item()
    assert math.isclose(pm.forward(g, m), z, rel_tol=1e-5, abs_tol=1e-6)
    assert math.isclose(pm.predict_gflops(g, m), pm.denormalize_label(m, pm.forward(g, m)))


def test_sweeper_end_to_end_int64_and_int32_hosts(cuda_device, g_model):
    """Sweeper.run_host (pinned host indices read in place by the scorer, scores + top-k
    out) equals the device-resident sweep, for int64 and narrowed int32 indices."""
    m = device_model(g_model)
    spec = pk.KernelSpec("conv2d", 56, 64, 64, 3, 3, 1)
    space = pk.build_knob_space(spec)
    lay = _layout(spec, "super")
    sw = ps.Sweeper(m, spec, space, lay, 100_000, k=64)
    idx = torch.from_numpy(np.random.default_rng(11).integers(0, space.size, 99_999))
    ti, ts = sw.run_device(idx.cuda())
    z_dev, ti, ts = sw.z[:99_999].clone(), ti.clone(), ts.clone()
    for host in (idx.pin_memory(), idx.to(torch.int32).pin_memory()):
        z_h, ti_h, ts_h = sw.run_host(host)
        assert torch.equal(z_h, z_dev.cpu())
        assert torch.equal(ti_h, ti.cpu()) and torch.equal(ts_h, ts.cpu())
    # two steps in flight (alternating host result slots): each ticket keeps its own results
    other = torch.from_numpy(np.random.default_rng(12).integers(0, space.size, 50_000))
    t1 = sw.submit(idx.pin_memory())
    t2 = sw.submit(other.to(torch.int32).pin_memory())
    z2, ti2, _ = (x.clone() for x in sw.wait(t2))
    z1, ti1, _ = sw.wait(t1)
    assert torch.equal(z1, z_dev.cpu()) and torch.equal(ti1, ti.cpu())
    ti_o, _ = sw.run_device(other.cuda())
    assert torch.equal(z2, sw.z[:50_000].cpu()) and torch.equal(ti2, ti_o.cpu())
    # tickets are never reused: a consumed ticket is stale, a third step in flight is refused
    with pytest.raises(ps.DomainError):
        sw.wait(t1)
    t3 = sw.submit(idx.pin_memory())
    sw.submit(other.to(torch.int32).pin_memory())
    with pytest.raises(ps.DomainError):
        sw.submit(idx.pin_memory())
    assert t3 > t2 and torch.equal(sw.wait(t3)[1], ti.cpu())


def test_topk_refuses_indices_beyond_32_bits(cuda_device):
    z = torch.zeros(8, device="cuda")
    with pytest.raises(ps.DomainError):
        ps.topk(z, 4, torch.arange(8, device="cuda") + 2**32)
    with pytest.raises(ps.DomainError):
        ps.topk(z, 4, base=2**32 - 4)


def test_sweeper_fused_keys_match_score_topk(cuda_device, g_model):
    """The scorer-built (score, index) keys rank exactly like kt_topk over the scores
    (the exclusion-list path), for int64 / int32 / implicit indices, ties and padding."""
    m = device_model(g_model)
    spec = pk.KernelSpec("conv2d", 56, 64, 64, 3, 3, 1)
    space = pk.build_knob_space(spec)
    lay = _layout(spec, "super")
    sw = ps.Sweeper(m, spec, space, lay, 70_000, k=300)
    none = torch.empty(0, dtype=torch.int64, device="cuda")
    rng = np.random.default_rng(5)
    idx = rng.integers(0, space.size, 65_537)
    idx[100:400] = idx[7]  # duplicates: equal scores, the index breaks the tie
    d64 = torch.from_numpy(idx).cuda()
    ref_i, ref_s = (t.clone() for t in sw.run_device(d64, visited=none))
    z_ref = sw.z[:idx.size].clone()
    for arg in (d64, d64.to(torch.int32)):
        ti, ts = sw.run_device(arg)
        assert torch.equal(sw.z[:idx.size], z_ref)
        assert torch.equal(ti, ref_i) and torch.equal(ts, ref_s)
    ti, ts = sw.run_device(base=1000, count=5000)
    ri, rs = sw.run_device(torch.arange(1000, 6000, device="cuda"), visited=none)
    assert torch.equal(ti, ri) and torch.equal(ts, rs)
    z = ps.score_indices(m, spec, space, lay, idx)
    z = z.cpu().numpy() if isinstance(z, torch.Tensor) else np.asarray(z)
    order = np.lexsort((idx, -z.astype(np.float64)))[:300]
    assert np.array_equal(ref_i.cpu().numpy(), idx[order])


def test_sweeper_out_of_range_index_excluded(cuda_device, g_model):
    m = device_model(g_model)
    spec = pk.KernelSpec("conv2d", 56, 64, 64, 3, 3, 1)
    space = pk.build_knob_space(spec)
    sw = ps.Sweeper(m, spec, space, _layout(spec, "super"), 1000, k=8)
    idx = torch.arange(0, 1000, dtype=torch.int64)
    idx[3] = space.size + 5
    ti, _ = sw.run_device(idx.cuda())
    assert int(sw.err.item()) != 0 and torch.isnan(sw.z[3]) and space.size + 5 not in ti.tolist()
    sw.err.zero_()
    with pytest.raises(pg.DomainError):
        sw.run_host(idx.pin_memory())
    with pytest.raises(pg.DomainError):
        sw.run_host(torch.arange(10))  # not pinned


@pytest.mark.parametrize("dist", ["equal", "few", "nan", "normal"])
@pytest.mark.parametrize("n,k", [(1_000_003, 1024), (70_000, 1), (300, 512), (513, 512)])
def test_topk_adversarial_distributions(cuda_device, dist, n, k):
    """The one-kernel radix select on score distributions that stress its digit passes:
    all-equal scores (ties resolved on the index word), a handful of values, NaNs, and
    B <= k / B = k + 1; the workspace is reused across calls."""
    rng = np.random.default_rng(hash((dist, n, k)) % 2**32)
    if dist == "equal":
        z = np.full(n, 0.75, dtype=np.float32)
    elif dist == "few":
        z = rng.choice(np.array([-1.0, 0.0, 0.5, 3.0], dtype=np.float32), n)
    elif dist == "nan":
        z = rng.normal(size=n).astype(np.float32)
        z[rng.integers(0, n, n // 10)] = np.nan
    else:
        z = rng.normal(size=n).astype(np.float32)
    idx = rng.permutation(np.arange(10 * n, dtype=np.int64))[:n]
    zt, it = torch.from_numpy(z).cuda(), torch.from_numpy(idx).cuda()
    for _ in range(2):
        ti, ts = ps.topk(zt, k, it)
    key = np.where(np.isnan(z), np.inf, -z.astype(np.float64))  # NaN ranks last
    order = np.lexsort((idx, key))[: min(k, n)]
    got = ti.cpu().numpy()
    assert got[: min(k, n)].tolist() == idx[order].tolist()
    if k > n:
        assert (got[n:] == -1).all()
