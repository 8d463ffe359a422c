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


RNG_KEYS = (("golden-model",), ("sweep", 0), ("sweep", 7), ("metatrain", "super", 0), ("x", 1, 2.5, (1, "a"), True),
            ("bench-cfgs",), ("", -3, 1e-300))


@pytest.mark.parametrize("j", range(len(RNG_KEYS)))
def test_rng_from_matches_reference_stream(j):
    """Byte golden of the reference's rng_from streams (util.py:17-55; tests/golden/rng.npz)."""
    from paper_2102_04199_b200.util import rng_from, stable_digest
    from tests.conftest import load_golden

    g = load_golden("rng")
    key = RNG_KEYS[j]
    assert stable_digest(*key).encode() == g[f"k{j}/digest"].tobytes()
    r = rng_from(*key)
    assert r.bit_generator.random_raw(16).tobytes() == g[f"k{j}/raw"].tobytes()
    assert r.integers(0, 451_584_000, 8).tobytes() == g[f"k{j}/ints"].tobytes()
    assert r.normal(size=4).tobytes() == g[f"k{j}/normal"].tobytes()


# --- BASELINE.json configs (tests/golden/baseline.npz) ----------------------------------


@pytest.fixture(scope="module")
def g_base():
    from tests.conftest import load_golden

    return load_golden("baseline")


def _bench_conv2d(idx, rep):
    ext = ko.extents("conv2d", 56, 64, 64, 3, 3, 1)
    knobs = ko.knob_lists("conv2d", ext)
    adj, rows, mask = ko.layout("conv2d", rep == "super")
    ch = ko.decode([len(v) for _, v in knobs], idx)
    return ko.encode("conv2d", ext, knobs, ch, adj.shape[0], rows), adj, mask


@pytest.mark.parametrize("rep", ["raw", "super"])
def test_oracle_c1_scores_and_ranking_match_reference(g_base, rep):
    from tests._shared import expand_unique, rank_parity

    p = oracle_params(g_base)
    idx = g_base["c1/idx"]
    x, adj, mask = _bench_conv2d(idx, rep)
    u = ko.embed_batch(p, x, mask, adj)
    np.testing.assert_allclose(u, expand_unique(g_base, f"c1/{rep}/u"), rtol=1e-12, atol=1e-12)
    z = ko.head_forward_batch(u, p["head_w"], p["head_b"])
    np.testing.assert_allclose(z, g_base[f"c1/{rep}/z"], rtol=1e-12, atol=1e-12)
    top = ko.rank_history(idx, z, set(), 512)
    assert top == g_base[f"c1/{rep}/top"].tolist()
    assert rank_parity(top, g_base[f"c1/{rep}/top"], idx, g_base[f"c1/{rep}/z"])["exact"]


def test_c5_indices_regenerate_from_rng(g_base):
    from paper_2102_04199_b200.kernels import KernelSpec, build_knob_space
    from tests._shared import sweep_indices

    n = int(g_base["c5/n"])
    idx = sweep_indices(n, build_knob_space(KernelSpec("conv2d", 56, 64, 64, 3, 3, 1)).size)
    assert len(np.unique(idx)) == n
    assert idx.sum() == g_base["c5/idx_sum"][0]
    assert (idx * np.arange(n)).sum() % (1 << 61) == g_base["c5/idx_sum"][1]
    assert set(g_base["c5/top"].tolist()) <= set(idx.tolist())


def test_oracle_c2_grad_matches_reference(g_base):
    """Batch-512 mixed-op super gradient (kink-free set) through the oracle."""
    from paper_2102_04199_b200.kernels import OP_TYPES

    p = oracle_params(g_base)
    key = "c2/super/kf"
    trip = []
    for op_i, i in zip(g_base[f"{key}/op"], g_base[f"{key}/idx"]):
        op = ("conv2d", "winograd", "depthwise")[int(op_i)]
        assert op in OP_TYPES
        ext = ko.extents(op, 56, 64, 64, 3, 3, 1)
        knobs = ko.knob_lists(op, ext)
        adj, rows, mask = ko.layout(op, True)
        ch = ko.decode([len(v) for _, v in knobs], np.array([i]))
        trip.append((ko.encode(op, ext, knobs, ch, adj.shape[0], rows)[0], adj, mask))
    loss, g = ko.grad(p, trip, g_base[f"{key}/label"].tolist())
    assert abs(loss - float(g_base[f"{key}/loss"])) <= 1e-12 * loss
    flat = np.concatenate([a.ravel() for a in g["gcn"] + [g["agg"]] + [
        t for w, b in zip(g["head_w"], g["head_b"]) for t in (w, b)]])
    np.testing.assert_allclose(flat, g_base[f"{key}/grad"], rtol=1e-9, atol=1e-13)


def test_rank_parity_helper():
    from tests._shared import rank_parity

    idx = np.arange(10)
    z = np.array([5.0, 5.0, 4.0, 3.0, 3.0 + 1e-7, 2.0, 1.0, 1.0, 0.5, 0.0])
    ref = ko.rank_history(idx, z, set(), 5)
    assert ref == [0, 1, 2, 4, 3]
    assert rank_parity(ref, ref, idx, z) == {"exact": True, "hard_flips": 0, "tie_flips": 0, "near_flips": 0,
                                            "max_flip_gap": 0.0}
    r = rank_parity([0, 1, 2, 3, 4], ref, idx, z)  # near tie (gap 1e-7 < 1e-5 * 3)
    assert not r["exact"] and r["hard_flips"] == 0 and r["near_flips"] == 1
    r = rank_parity([1, 0, 2, 4, 3], ref, idx, z)  # exact-tie class out of index order
    assert r["hard_flips"] == 0 and r["tie_flips"] == 1 and r["near_flips"] == 0
    r = rank_parity([0, 1, 4, 3, 5], ref, idx, z)  # dropped 2 (score 4) for 5 (score 2)
    assert r["hard_flips"] >= 3
