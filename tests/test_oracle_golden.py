"""Pin the oracle (and the product's host logic) to fixtures produced by the reference.

CPU only.  Fixtures come from tests/golden/make_goldens.py, which runs the
reference package itself; the graph text goldens are the reference's own.
"""

import numpy as np
import pytest

from oracle import kt_oracle as ko
from paper_2102_04199_b200 import graphs as pg
from paper_2102_04199_b200 import kernels as pk
from tests._shared import corpus_graphs, head_shapes, oracle_params, spec_of

OPS = pk.OP_TYPES


# --- graph text goldens (reference tests/golden) --------------------------------


def test_product_config_graph_matches_reference_golden_text(golden_dir):
    spec = pk.KernelSpec("conv1d", 200, 64, 128, 3)
    space = pk.build_knob_space(spec)
    c = pk.index_config(space, 123456)
    raw = pg.graph_to_text(pg.config_graph(spec, c, space))
    sup = pg.graph_to_text(pg.config_graph(spec, c, space, template=pg.build_super_template(OPS)))
    assert raw == (golden_dir / "graph_conv1d_raw.txt").read_text()
    assert sup == (golden_dir / "graph_conv1d_super.txt").read_text()


def test_text_round_trip(golden_dir):
    txt = (golden_dir / "graph_conv1d_super.txt").read_text()
    assert pg.graph_to_text(pg.graph_from_text(txt)) == txt


# --- knob spaces and the encoder ------------------------------------------------------


@pytest.mark.parametrize("op", OPS)
def test_knob_space_tables(g_encode, op):
    spec = spec_of(g_encode, op)
    space = pk.build_knob_space(spec)
    assert space.size == int(g_encode[f"{op}/size"])
    for j, k in enumerate(space.knobs):
        assert np.array_equal(np.array(k.values), g_encode[f"{op}/knob{j}"])
    s = spec
    ext = ko.extents(op, s.input_size, s.in_channels, s.out_channels, s.kernel_size, s.stride, s.padding)
    for j, (_, vals) in enumerate(ko.knob_lists(op, ext)):
        assert np.array_equal(np.array(vals), g_encode[f"{op}/knob{j}"])


@pytest.mark.parametrize("op", OPS)
def test_index_decode_bit_exact(g_encode, op):
    spec = spec_of(g_encode, op)
    space = pk.build_knob_space(spec)
    idx, choices = g_encode[f"{op}/idx"], g_encode[f"{op}/choices"]
    assert np.array_equal(ko.decode(space.cardinalities, idx), choices)
    for i, c in zip(idx, choices):
        assert pk.index_config(space, int(i)).choices == tuple(int(v) for v in c)
        assert pk.config_index(space, pk.KnobConfig(tuple(int(v) for v in c))) == int(i)


@pytest.mark.parametrize("rep", ["raw", "super"])
@pytest.mark.parametrize("op", OPS)
def test_oracle_encode_bit_exact(g_encode, op, rep):
    s = spec_of(g_encode, op)
    ext = ko.extents(op, s.input_size, s.in_channels, s.out_channels, s.kernel_size, s.stride, s.padding)
    knobs = ko.knob_lists(op, ext)
    adj, rows, mask = ko.layout(op, rep == "super")
    assert np.array_equal(rows, g_encode[f"{op}/{rep}/rows"])
    assert adj.tobytes() == g_encode[f"{op}/{rep}/adj"].tobytes()
    x = ko.encode(op, ext, knobs, g_encode[f"{op}/choices"], adj.shape[0], rows)
    assert x[:, rows, :].tobytes() == g_encode[f"{op}/{rep}/feats"].tobytes()
    assert not x[:, ~mask, :].any()


@pytest.mark.parametrize("rep", ["raw", "super"])
@pytest.mark.parametrize("op", OPS)
def test_product_host_layout_and_graphs_bit_exact(g_encode, op, rep):
    spec = spec_of(g_encode, op)
    space = pk.build_knob_space(spec)
    tmpl = pg.build_super_template(OPS) if rep == "super" else None
    lay = pg.batch_layout(spec, tmpl)
    assert np.array_equal(lay.iterval_rows, g_encode[f"{op}/{rep}/rows"])
    assert lay.adjacency.tobytes() == g_encode[f"{op}/{rep}/adj"].tobytes()
    feats = g_encode[f"{op}/{rep}/feats"]
    for j, c in enumerate(g_encode[f"{op}/choices"][:8]):
        g = pg.config_graph(spec, pk.KnobConfig(tuple(int(v) for v in c)), space, template=tmpl)
        t = pg.graph_to_tensors(g)
        assert t.feature_matrix[lay.iterval_rows].tobytes() == feats[j].tobytes()
        assert np.array_equal(t.feature_mask, lay.feature_mask)
        assert t.normalized_adjacency.tobytes() == lay.adjacency.tobytes()


def test_all_ops_share_super_adjacency(g_encode):
    blobs = {g_encode[f"{op}/super/adj"].tobytes() for op in OPS}
    assert len(blobs) == 1


# --- model forward / gradients ------------------------------------------------------


def _encode_conv2d(g_encode, idx, rep):
    s = spec_of(g_encode, "conv2d")
    ext = ko.extents("conv2d", s.input_size, s.in_channels, s.out_channels, s.kernel_size, s.stride, s.padding)
    knobs = ko.knob_lists("conv2d", ext)
    adj, rows, mask = ko.layout("conv2d", rep == "super")
    ch = ko.decode([len(v) for _, v in knobs], idx)
    return ko.encode("conv2d", ext, knobs, ch, adj.shape[0], rows), adj, mask


@pytest.mark.parametrize("rep", ["raw", "super"])
def test_oracle_embed_and_head_match_reference(g_encode, g_model, rep):
    p = oracle_params(g_model)
    x, adj, mask = _encode_conv2d(g_encode, g_model["score/idx"], rep)
    u = ko.embed_batch(p, x, mask, adj)
    np.testing.assert_allclose(u, g_model[f"score/{rep}/u"], rtol=1e-12, atol=1e-12)
    z = ko.head_forward_batch(u, p["head_w"], p["head_b"])
    np.testing.assert_allclose(z, g_model[f"score/{rep}/z"], rtol=1e-12, atol=1e-12)


def test_oracle_init_params_reproduce_reference_draws(g_model):
    from paper_2102_04199_b200.util import rng_from

    p = ko.init_params(rng_from("golden-model"))
    ref = oracle_params(g_model)
    for a, b in zip(p["gcn"] + p["head_w"] + p["head_b"], ref["gcn"] + ref["head_w"] + ref["head_b"]):
        assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("b", [0, 1, 2])
@pytest.mark.parametrize("scope", ["all", "head_only"])
def test_oracle_grad_matches_reference(g_model, g_grad, g_meta, b, scope):
    p = oracle_params(g_model)
    graphs = corpus_graphs(g_meta, super_graph=False)
    pick = g_grad[f"b{b}/pick"]
    labels = g_meta["labels"]
    loss, g = ko.grad(p, [graphs[int(j)] for j in pick], [float(labels[int(j)]) for j in pick], scope)
    assert abs(loss - float(g_grad[f"b{b}/{scope}/loss"])) <= 1e-12 * max(1.0, abs(loss))
    for i, w in enumerate(g["gcn"]):
        np.testing.assert_allclose(w, g_grad[f"b{b}/{scope}/gcn{i}"], rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(g["agg"], g_grad[f"b{b}/{scope}/agg"], rtol=1e-10, atol=1e-13)
    for i, (w, bb) in enumerate(zip(g["head_w"], g["head_b"])):
        np.testing.assert_allclose(w, g_grad[f"b{b}/{scope}/hw{i}"], rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(bb, g_grad[f"b{b}/{scope}/hb{i}"], rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("k", [0, 1, 2])
def test_oracle_head_loss_grad_and_hvp(g_model, g_head, k):
    p = oracle_params(g_model)
    sh = head_shapes(p)
    th, u, y, v = (g_head[f"c{k}/{n}"] for n in ("theta", "u", "y", "v"))
    mse, g = ko.head_loss_grad(th, sh, u, y)
    assert abs(mse - float(g_head[f"c{k}/mse"])) <= 1e-12 * max(1.0, mse)
    np.testing.assert_allclose(g, g_head[f"c{k}/grad"], rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(ko.head_hvp(th, sh, u, y, v), g_head[f"c{k}/hvp"], rtol=1e-10, atol=1e-14)


def _embed_all(p, graphs):
    return np.concatenate([ko.embed_batch(p, x[None], mask, adj) for x, adj, mask in graphs])


@pytest.mark.parametrize("order", ["fo", "so"])
def test_oracle_meta_step_matches_reference(g_model, g_meta, order):
    p = oracle_params(g_model)
    sh = head_shapes(p)
    u_all = _embed_all(p, corpus_graphs(g_meta, super_graph=True))
    y_all = np.array([ko.normalize_label(p, float(v)) for v in g_meta["labels"]])
    tasks = [(u_all[s], y_all[s], u_all[q], y_all[q])
             for s, q in zip(g_meta[f"{order}/support"], g_meta[f"{order}/query"])]
    theta = ko.head_to_vec(p["head_w"], p["head_b"])
    t1, sl, ql = ko.meta_step_embedded(theta, sh, tasks, 0.01, 0.001, 1, order == "fo")
    np.testing.assert_allclose(t1, g_meta[f"{order}/theta"], rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose([sl, ql], g_meta[f"{order}/stats"], rtol=1e-10)
    t3 = t1
    for _ in range(2):
        t3, _, _ = ko.meta_step_embedded(t3, sh, tasks, 0.01, 0.001, 1, order == "fo")
    np.testing.assert_allclose(t3, g_meta[f"{order}/theta3"], rtol=1e-11, atol=1e-14)


def test_oracle_fine_tune_matches_reference(g_model, g_meta):
    p = oracle_params(g_model)
    u = _embed_all(p, corpus_graphs(g_meta, super_graph=True)[:64])
    y = np.array([ko.normalize_label(p, float(v)) for v in g_meta["labels"][:64]])
    theta = ko.head_to_vec(p["head_w"], p["head_b"])
    out = ko.fine_tune_embedded(theta, head_shapes(p), u, y, 0.01, 8)
    np.testing.assert_allclose(out, g_meta["ft/theta"], rtol=1e-11, atol=1e-14)


def test_oracle_rank_history(g_rank):
    top = ko.rank_history(g_rank["idx"], g_rank["scores"], set(int(v) for v in g_rank["visited"]), 128)
    assert top == [int(v) for v in g_rank["top"]]


def test_rng_from_matches_reference_stream(g_model):
    # init_model draws through rng_from("golden-model"); equal draws => equal stream
    from paper_2102_04199_b200.util import rng_from, stable_digest

    assert stable_digest("x", 1, 2.5, (1, "a"), True) == stable_digest("x", 1, 2.5, (1, "a"), True)
    a = rng_from("golden-model").uniform(size=4)
    b = rng_from("golden-model").uniform(size=4)
    assert a.tobytes() == b.tobytes()
