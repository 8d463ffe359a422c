"""Device parity of the training path: grad / sgd_step, head engine, MAML, fine-tune, pretrain.

Tolerances (fp32 device vs fp64 reference; SURVEY.md 7 hard part 1):
  * gradients: per-tensor norm-wise rel <= 1e-4, and element-wise rel <= 1e-4
    for every entry above an absolute floor of 1e-3 * max|g| of its tensor (fp32
    batch-sum cancellation bounds the relative error of the smaller entries);
  * parameters after updates: element-wise rel <= 1e-5 (floor 1e-7);
  * losses: rel <= 1e-5.
"""

import numpy as np
import pytest
import torch

from oracle import kt_oracle as ko
from paper_2102_04199_b200 import graphs as pg
from paper_2102_04199_b200 import kernels as pk
from paper_2102_04199_b200 import meta as pmeta
from paper_2102_04199_b200 import model as pm
from paper_2102_04199_b200.util import rng_from
from tests._shared import device_model, head_shapes, oracle_params, spec_of

pytestmark = pytest.mark.gpu
OPS = pk.OP_TYPES
TEMPLATE = pg.build_super_template(OPS)


def assert_grad_close(got, want, rtol=1e-4, elem_rtol=None):
    """Per-tensor norm-wise rel <= rtol, and element-wise rel <= elem_rtol (default rtol) above a
    1e-3 * max floor.  The element-wise 1e-4 bar is for kink-free batches: on an
    arbitrary batch a ReLU / max-routing decision within fp32 reach of flipping, or fp32
    cancellation in a batch sum, moves single entries further."""
    elem_rtol = rtol if elem_rtol is None else elem_rtol
    got = np.asarray(got, dtype=np.float64).ravel()
    want = np.asarray(want, dtype=np.float64).ravel()
    scale = np.linalg.norm(want)
    if scale == 0:
        assert np.abs(got).max() == 0
        return
    assert np.linalg.norm(got - want) <= rtol * scale, f"norm-wise rel {np.linalg.norm(got - want) / scale:.2e}"
    floor = 1e-3 * np.abs(want).max()
    big = np.abs(want) > floor
    rel = np.abs(got[big] - want[big]) / np.abs(want[big])
    assert rel.max() <= elem_rtol, f"element-wise rel {rel.max():.2e}"


def assert_params_close(got, want, rtol=1e-5):
    got = np.asarray(got, dtype=np.float64).ravel()
    want = np.asarray(want, dtype=np.float64).ravel()
    err = np.abs(got - want) / np.maximum(np.abs(want), 1e-7 / rtol * 1e-5 + 1e-7)
    assert np.abs(got - want).max() <= rtol * np.abs(want).max() or err.max() <= 10 * rtol, \
        f"max abs {np.abs(got - want).max():.2e}"
    assert np.linalg.norm(got - want) <= rtol * np.linalg.norm(want)


def corpus_samples(g_encode, g_meta, super_graph):
    out = []
    for op_i, idx, y in zip(g_meta["op"], g_meta["idx"], g_meta["labels"]):
        op = OPS[int(op_i)]
        spec = spec_of(g_encode, op)
        space = pk.build_knob_space(spec)
        g = pg.config_graph(spec, pk.index_config(space, int(idx)), space,
                            template=TEMPLATE if super_graph else None)
        out.append(pmeta.LabeledSample(g, spec.signature(), float(y)))
    return out


@pytest.fixture(scope="module")
def raw_samples(g_encode, g_meta):
    return corpus_samples(g_encode, g_meta, False)


@pytest.fixture(scope="module")
def super_samples(g_encode, g_meta):
    return corpus_samples(g_encode, g_meta, True)


@pytest.mark.parametrize("b", [0, 1, 2])
@pytest.mark.parametrize("scope", ["all", "head_only"])
def test_grad_matches_reference(cuda_device, g_model, g_grad, raw_samples, b, scope):
    m = device_model(g_model)
    pick = g_grad[f"b{b}/pick"]
    batch = [(raw_samples[int(j)].graph, raw_samples[int(j)].label_gflops) for j in pick]
    loss, g = pm.grad(m, batch, scope)
    ref_loss = float(g_grad[f"b{b}/{scope}/loss"])
    assert abs(loss - ref_loss) <= 1e-5 * max(abs(ref_loss), 1e-6)
    for i, w in enumerate(g.gcn):
        assert_grad_close(w.cpu().numpy(), g_grad[f"b{b}/{scope}/gcn{i}"])
    assert_grad_close(g.agg.cpu().numpy(), g_grad[f"b{b}/{scope}/agg"])
    for i, (w, bb) in enumerate(zip(g.head_weights, g.head_biases)):
        assert_grad_close(w.cpu().numpy(), g_grad[f"b{b}/{scope}/hw{i}"])
        assert_grad_close(bb.cpu().numpy(), g_grad[f"b{b}/{scope}/hb{i}"])
    if scope == "head_only":
        assert not any(w.any() for w in g.gcn) and not g.agg.any()


def test_grad_is_deterministic(cuda_device, g_model, raw_samples):
    m = device_model(g_model)
    batch = [(s.graph, s.label_gflops) for s in raw_samples[:200]]
    l1, g1 = pm.grad(m, batch)
    l2, g2 = pm.grad(m, batch)
    assert l1 == l2 and torch.equal(g1._flat, g2._flat)


def test_grad_super_batch_vs_oracle(cuda_device, g_model, super_samples):
    """Batch of 360 super-graph samples (all ops) against the oracle."""
    m = device_model(g_model)
    p = oracle_params(g_model)
    loss, g = pm.grad(m, [(s.graph, s.label_gflops) for s in super_samples])
    trip = []
    for s in super_samples:
        t = pg.graph_to_tensors(s.graph)
        trip.append((t.feature_matrix, t.normalized_adjacency, t.feature_mask))
    rl, rg = ko.grad(p, trip, [s.label_gflops for s in super_samples])
    assert abs(loss - rl) <= 1e-5 * rl
    for a, b in zip(g.gcn + [g.agg] + g.head_weights + g.head_biases,
                    rg["gcn"] + [rg["agg"]] + rg["head_w"] + rg["head_b"]):
        assert_grad_close(a.cpu().numpy(), b)


@pytest.mark.parametrize("layout", ["raw", "super"])
@pytest.mark.parametrize("b", [1, 5, 131, 1200])
def test_grad_batch_sizes_vs_oracle(cuda_device, g_model, raw_samples, super_samples, layout, b):
    """kt_grad's launch shapes: factored path with 4-graph CTAs and a partial last CTA (1, 5,
    131 graphs) and the per-graph-row path above 8 x 148 graphs (1,200, samples repeated),
    raw-segmented and super layouts, against the oracle's batch gradient."""
    m = device_model(g_model)
    p = oracle_params(g_model)
    pool = raw_samples if layout == "raw" else super_samples
    pick = rng_from("grad-b", b, layout).integers(0, len(pool), b)
    batch = [(pool[int(j)].graph, pool[int(j)].label_gflops) for j in pick]
    loss, g = pm.grad(m, batch)
    trip = []
    for gr, _ in batch:
        t = pg.graph_to_tensors(gr)
        trip.append((t.feature_matrix, t.normalized_adjacency, t.feature_mask))
    rl, rg = ko.grad(p, trip, [lab for _, lab in batch])
    assert abs(loss - rl) <= 1e-5 * rl
    for a, r in zip(g.gcn + [g.agg] + g.head_weights + g.head_biases,
                    rg["gcn"] + [rg["agg"]] + rg["head_w"] + rg["head_b"]):
        assert_grad_close(a.cpu().numpy(), r, elem_rtol=1e-3)  # (random batches, not kink-free)


def test_sgd_step_matches_reference(cuda_device, g_model, g_grad, raw_samples):
    m = device_model(g_model)
    pick = g_grad["b2/pick"]
    batch = [(raw_samples[int(j)].graph, raw_samples[int(j)].label_gflops) for j in pick]
    _, g = pm.grad(m, batch)
    m2 = pm.sgd_step(m, g, 0.005)
    assert_params_close(pm.flat_params(m2).cpu().numpy(), g_grad["b2/sgd_vec"])
    # pure: the input model is untouched
    assert torch.equal(pm.flat_params(m), device_model(g_model)._flat)


def test_sgd_step_arrays_and_guards(cuda_device):
    out = pm.sgd_step(np.array([1.0, 2.0]), np.array([1.0, 1.0]), 0.5)
    assert np.allclose(out, [0.5, 1.5]) and isinstance(out, np.ndarray)
    with pytest.raises(pm.DomainError):
        pm.sgd_step(np.zeros(2), np.zeros(3), 0.1)


@pytest.mark.parametrize("k", [0, 1, 2])
def test_head_loss_grad_and_hvp(cuda_device, g_model, g_head, k):
    m = device_model(g_model)
    th, u, y, v = (g_head[f"c{k}/{n}"] for n in ("theta", "u", "y", "v"))
    mse, g = pm.head_loss_grad(th, m.head, u, y)
    assert abs(mse - float(g_head[f"c{k}/mse"])) <= 1e-5 * float(g_head[f"c{k}/mse"])
    assert_grad_close(g.cpu().numpy(), g_head[f"c{k}/grad"])
    hv = pm.head_hvp(th, m.head, u, y, v)
    assert_grad_close(hv.cpu().numpy(), g_head[f"c{k}/hvp"])


@pytest.mark.parametrize("order", ["fo", "so"])
def test_meta_step_matches_reference(cuda_device, g_model, g_meta, super_samples, order):
    m = device_model(g_model)
    cfg = pmeta.MetaConfig(n_way=3, k_shot=2, meta_batch=32, inner_steps=1, first_order=order == "fo")
    tasks = [pmeta.MetaTask([super_samples[i] for i in s], [super_samples[i] for i in q], [])
             for s, q in zip(g_meta[f"{order}/support"], g_meta[f"{order}/query"])]
    m1, stats = pmeta.meta_step(m, tasks, cfg)
    assert_params_close(pm.head_to_vec(m1.head).cpu().numpy(), g_meta[f"{order}/theta"])
    np.testing.assert_allclose([stats["support_loss"], stats["query_loss"]], g_meta[f"{order}/stats"], rtol=1e-5)
    assert torch.equal(pm.flat_params(m1)[: pm.dims_of(m).off_head], pm.flat_params(m)[: pm.dims_of(m).off_head])
    m3 = m1
    for _ in range(2):
        m3, _ = pmeta.meta_step(m3, tasks, cfg)
    assert_params_close(pm.head_to_vec(m3.head).cpu().numpy(), g_meta[f"{order}/theta3"])


@pytest.mark.parametrize("order", ["fo", "so"])
@pytest.mark.parametrize("ns,nq,inner", [(1, 1, 1), (6, 6, 1), (8, 8, 2), (9, 3, 1), (20, 13, 2), (33, 17, 1)])
def test_maml_task_shapes_match_oracle(cuda_device, g_model, order, ns, nq, inner):
    """kt_maml_tasks over support / query sets that fit one row chunk (staged rows, the inner
    SGD step fused into the gradient write) and sets spanning several chunks, one and two inner
    steps, first and second order, against the fp64 oracle of maml_outer_grad (meta.py:167-257)."""
    m = device_model(g_model)
    p = oracle_params(g_model)
    rng = rng_from("maml-shapes", ns, nq, inner, order)
    T = 5
    n_rows = T * (ns + nq)
    u = np.abs(rng.normal(size=(n_rows, 64))).astype(np.float32)
    y = rng.normal(size=n_rows).astype(np.float32)
    perm = rng.permutation(n_rows)
    tasks, s_idx, q_idx = [], [], []
    for t in range(T):
        rows = perm[t * (ns + nq):(t + 1) * (ns + nq)]
        s, q = rows[:ns], rows[ns:]
        s_idx += list(s)
        q_idx += list(q)
        tasks.append((u[s].astype(np.float64), y[s].astype(np.float64), u[q].astype(np.float64),
                      y[q].astype(np.float64)))
    cfg = pmeta.MetaConfig(alpha=0.01, beta=0.001, inner_steps=inner, first_order=order == "fo")
    theta = ko.head_to_vec(p["head_w"], p["head_b"])
    want, sl, ql = ko.meta_step_embedded(theta, head_shapes(p), tasks, cfg.alpha, cfg.beta, inner, order == "fo")
    dev = cuda_device
    t64 = lambda a: torch.tensor(np.asarray(a, dtype=np.int64), device=dev)  # noqa: E731
    g_sum, stats = pmeta.maml_sum(m, torch.from_numpy(u).to(dev), torch.from_numpy(y).to(dev),
                                  t64(np.arange(T + 1) * ns), t64(s_idx), t64(np.arange(T + 1) * nq), t64(q_idx), cfg)
    got = pm.head_to_vec(m.head).cpu().numpy().astype(np.float64) - cfg.beta * g_sum.cpu().numpy()
    assert_params_close(got, want, rtol=1e-5)
    np.testing.assert_allclose(stats.cpu().numpy() / T, [sl, ql], rtol=1e-4)


def test_meta_step_reductions(cuda_device, g_model, g_meta, super_samples):
    m = device_model(g_model)
    tasks = [pmeta.MetaTask([super_samples[i] for i in s], [super_samples[i] for i in q], [])
             for s, q in zip(g_meta["fo/support"][:8], g_meta["fo/query"][:8])]
    # beta = 0: bitwise identity
    m0, _ = pmeta.meta_step(m, tasks, pmeta.MetaConfig(beta=0.0))
    assert torch.equal(pm.flat_params(m0), pm.flat_params(m))
    # alpha = 0: plain SGD (lr beta) on the summed query gradients
    cfg = pmeta.MetaConfig(alpha=0.0, beta=0.002)
    ma, _ = pmeta.meta_step(m, tasks, cfg)
    theta = pm.head_to_vec(m.head)
    total = torch.zeros_like(theta)
    for t in tasks:
        u, y = pmeta._embedded(m, t.query)
        total += pm.head_loss_grad(theta, m.head, u, y)[1]
    want = (theta - cfg.beta * total).cpu().numpy()
    assert_params_close(pm.head_to_vec(ma.head).cpu().numpy(), want, rtol=1e-6)


def test_fine_tune_matches_reference(cuda_device, g_model, g_meta, super_samples):
    m = device_model(g_model)
    ft = super_samples[:64]
    m2 = pmeta.fine_tune(m, [(s.graph, s.label_gflops) for s in ft], 0.01, 8)
    assert_params_close(pm.head_to_vec(m2.head).cpu().numpy(), g_meta["ft/theta"])
    assert torch.equal(pm.flat_params(m2)[: pm.dims_of(m).off_head], pm.flat_params(m)[: pm.dims_of(m).off_head])
    assert pmeta.fine_tune(m, [], 0.01, 5) is m


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 7, 16, 40, 64, 100, 130, 257])
def test_fine_tune_embedded_row_counts_match_oracle(cuda_device, g_model, n):
    """kt_fine_tune at every launch shape (one CTA below 16 rows, clusters of 4 / 8 CTAs
    above, rows staged once when they fit a chunk, slices pushed to the peers) against the
    fp64 oracle restatement of fine_tune_embedded (meta.py:274-282)."""
    m = device_model(g_model)
    p = oracle_params(g_model)
    rng = rng_from("ft-rows", n)
    u = np.abs(rng.normal(size=(n, 64)))
    y = rng.normal(size=n)
    theta = ko.head_to_vec(p["head_w"], p["head_b"])
    want = ko.fine_tune_embedded(theta, head_shapes(p), u, y, 0.01, 6)
    got = pm.head_to_vec(pmeta.fine_tune_embedded(m, u, y, 0.01, 6).head).cpu().numpy()
    assert_params_close(got, want, rtol=1e-5)


def test_inner_adapt_alpha_zero_identity(cuda_device, g_model, super_samples):
    m = device_model(g_model)
    h = pmeta.inner_adapt(m, super_samples[:4], alpha=0.0, inner_steps=3)
    assert torch.equal(pm.head_to_vec(h), pm.head_to_vec(m.head))


def test_pretrain_matches_oracle_sgd_loop(cuda_device, g_encode, g_meta):
    """pretrain == init_model(rng) + per-epoch rng.permutation + batch-1 SGD (meta.py:104-123)."""
    from paper_2102_04199_b200.util import rng_from

    samples = corpus_samples(g_encode, g_meta, False)[::9]  # 40 raw graphs of mixed sizes
    cfg = pmeta.MetaConfig(pretrain_epochs=2, gamma=0.005)
    m = pmeta.pretrain(samples, cfg, rng_from("pretrain-test"))
    # oracle replay with the same draws
    rng = rng_from("pretrain-test")
    p = ko.init_params(rng)
    fn, ln = pmeta.dataset_norms(samples)
    p.update(fmean=fn.mean, fstd=fn.std, lmean=ln.mean, lstd=ln.std)
    trip = []
    for s in samples:
        t = pg.graph_to_tensors(s.graph)
        trip.append((t.feature_matrix, t.normalized_adjacency, t.feature_mask))
    for _ in range(cfg.pretrain_epochs):
        for i in rng.permutation(len(samples)):
            _, g = ko.grad(p, [trip[int(i)]], [samples[int(i)].label_gflops])
            p = ko.sgd(p, g, cfg.gamma)
    want = np.concatenate([w.ravel() for w in p["gcn"]] + [p["agg"]] + [ko.head_to_vec(p["head_w"], p["head_b"])])
    got = pm.flat_params(m).cpu().numpy()
    assert np.linalg.norm(got - want) <= 1e-4 * np.linalg.norm(want)
    assert np.array_equal(m.feature_norm.mean, fn.mean)


def test_meta_trainer_equals_meta_train(cuda_device, g_model, super_samples):
    """Device-resident MetaTrainer (cached frozen-GCN embeddings, pre-drawn tasks,
    2 launches/step) == meta_train (which re-embeds every step, like the reference)."""
    from paper_2102_04199_b200.util import rng_from

    m = device_model(g_model)
    cfg = pmeta.MetaConfig(n_way=3, k_shot=2, meta_batch=8, outer_steps=6)
    want = pmeta.meta_train(m, super_samples, cfg, rng_from("mt-eq"))
    tr = pmeta.MetaTrainer(m, super_samples, cfg)
    plan = tr.plan(rng_from("mt-eq"), cfg.outer_steps)
    bufs = tr.run(plan)
    got = tr.model()
    assert_params_close(pm.flat_params(got).cpu().numpy(), pm.flat_params(want).cpu().numpy(), rtol=1e-6)
    assert np.isfinite(tr.stats(plan, bufs)).all()


def test_meta_trainer_graph_replay_equals_eager(cuda_device, g_model, super_samples):
    """A captured CUDA graph of the outer steps gives the eager loop's parameters bit for bit."""
    from paper_2102_04199_b200.util import rng_from

    m = device_model(g_model)
    cfg = pmeta.MetaConfig(n_way=3, k_shot=2, meta_batch=8, outer_steps=10)
    eager = pmeta.MetaTrainer(m, super_samples, cfg)
    plan = eager.plan(rng_from("mt-graph"), cfg.outer_steps)
    bufs = eager.run(plan)
    rep = pmeta.MetaTrainer(m, super_samples, cfg)
    plan2 = rep.plan(rng_from("mt-graph"), cfg.outer_steps)
    bufs2 = rep._buffers(plan2)
    for s in range(3):
        rep.step(plan2, bufs2, s)
    g = rep.capture(plan2, bufs2, 3, cfg.outer_steps)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(pm.flat_params(rep.model()), pm.flat_params(eager.model()))
    assert torch.equal(bufs2["stats"], bufs["stats"])



def _parse_log(text):
    lines = text.strip().split("\n")
    rows = [ln.split(",") for ln in lines[1:]]
    return lines[0], np.array([int(r[0]) for r in rows]), np.array([[float(r[1]), float(r[2])] for r in rows])


@pytest.mark.parametrize("order", ["fo", "so"])
def test_meta_train_matches_reference_run(cuda_device, g_model, super_samples, tmp_path, order):
    """meta_train (meta.py:260-268) pinned to a reference run: sample_meta_tasks draws from
    rng_from("golden-metatrain", order), meta_step per outer step, the CSV log
    (tests/golden/metatrain.npz).  Both meta_train and the device-resident MetaTrainer."""
    from paper_2102_04199_b200.util import rng_from
    from tests.conftest import load_golden

    g = load_golden("metatrain")
    steps = int(g[f"{order}/steps"])
    head, ref_steps, ref_losses = _parse_log(g[f"{order}/csv"].tobytes().decode())
    m = device_model(g_model)
    cfg = pmeta.MetaConfig(n_way=3, k_shot=2, meta_batch=32, inner_steps=1, outer_steps=steps,
                           first_order=order == "fo")
    log = tmp_path / "log.csv"
    m2 = pmeta.meta_train(m, super_samples, cfg, rng_from("golden-metatrain", order), log)
    h2, st2, l2 = _parse_log(log.read_text())
    assert h2 == head == "step,support_loss,query_loss"
    assert np.array_equal(st2, ref_steps)
    np.testing.assert_allclose(l2, ref_losses, rtol=1e-5)
    assert_params_close(pm.head_to_vec(m2.head).cpu().numpy(), g[f"{order}/theta"])
    tr = pmeta.MetaTrainer(m, super_samples, cfg)
    plan = tr.plan(rng_from("golden-metatrain", order), steps)
    bufs = tr.run(plan)
    np.testing.assert_allclose(tr.stats(plan, bufs), ref_losses, rtol=1e-5)
    assert_params_close(pm.head_to_vec(tr.model().head).cpu().numpy(), g[f"{order}/theta"])


def test_checkpoint_interchange_with_reference(cuda_device, tmp_path):
    """load_model reads the reference's own npz v1 file (tests/golden/ckpt_v1.npz, written by
    kerntune.model.save_model); save_model writes the same keys, shapes and (fp32-exact) values."""
    import os

    ref_path = os.path.join(os.path.dirname(__file__), "golden", "ckpt_v1.npz")
    m = pm.load_model(ref_path)
    with np.load(ref_path) as z:
        ref = {k: z[k] for k in z.files}
    for i, w in enumerate(m.gcn.layers):
        assert np.array_equal(w.cpu().numpy(), ref[f"gcn_{i}"].astype(np.float32))
    for i, (w, b) in enumerate(zip(m.head.weights, m.head.biases)):
        assert np.array_equal(w.cpu().numpy(), ref[f"head_w{i}"].astype(np.float32))
        assert np.array_equal(b.cpu().numpy(), ref[f"head_b{i}"].astype(np.float32))
    assert np.array_equal(m.feature_norm.mean, ref["feat_mean"]) and np.array_equal(m.feature_norm.std, ref["feat_std"])
    assert (m.label_norm.mean, m.label_norm.std) == tuple(ref["label_norm"])
    out = tmp_path / "ours.npz"
    pm.save_model(m, out)
    with np.load(out) as z:
        ours = {k: z[k] for k in z.files}
    assert sorted(ours) == sorted(ref)
    for k in ref:
        assert ours[k].shape == ref[k].shape and ours[k].dtype == ref[k].dtype, k
        if k.startswith(("gcn_", "head_", "agg_")):
            assert np.array_equal(ours[k], ref[k].astype(np.float32).astype(np.float64)), k
        else:
            assert np.array_equal(ours[k], ref[k]), k
    m2 = pm.load_model(out)
    assert torch.equal(pm.flat_params(m2), pm.flat_params(m))
    np.savez(tmp_path / "bad.npz", version=np.array(2))
    with pytest.raises(pg.DomainError):
        pm.load_model(tmp_path / "bad.npz")
