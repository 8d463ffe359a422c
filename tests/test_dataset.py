"""Index-based datasets (harness.py:97-252 -> paper_2102_04199_b200.dataset).

CPU: load_records reads the reference's own save_dataset output (tests/golden/dataset/,
written by the reference) and reproduces its manifest content hash; tampering is
caught like load_dataset does.
GPU: IndexedDataset (device encode + array-built CSR) equals pack_graphs over the
reference-style materialised graphs; dataset_norms, grad_indexed and pretrain on it
match the reference's values on dataset_samples (tests/golden/dataset.npz).
"""

import os
import shutil

import numpy as np
import pytest

from paper_2102_04199_b200 import dataset as pd
from paper_2102_04199_b200.errors import ConfigError, DomainError

DS_DIR = os.path.join(os.path.dirname(__file__), "golden", "dataset")


def test_load_records_matches_reference_manifest(g_dataset):
    params, entries = pd.load_records(DS_DIR)
    assert params["n_kernels"] == len(entries) == 7
    assert sum(e.indices.size for e in entries) == g_dataset["raw/labels"].size
    labels = np.concatenate([np.maximum(e.gflops, 1e-3) for e in entries])
    assert np.array_equal(labels, g_dataset["raw/labels"])
    classes = [pd._spec_signature(e.spec) for e in entries for _ in range(e.indices.size)]
    assert classes == [str(c) for c in g_dataset["classes"]]


def test_load_records_rejects_tampering(tmp_path):
    d = tmp_path / "ds"
    shutil.copytree(DS_DIR, d)
    lines = (d / "samples.csv").read_text().splitlines()
    k, i, g, f = lines[1].split(",")
    lines[1] = ",".join([k, str(int(i) + 1), g, f])
    (d / "samples.csv").write_text("\n".join(lines) + "\n")
    with pytest.raises(ConfigError):
        pd.load_records(str(d))
    pd.load_records(str(d), verify=False)
    with pytest.raises(ConfigError):
        pd.load_records(str(tmp_path / "missing"))


# ---- device ---------------------------------------------------------------------------------

from tests.test_gpu_train import assert_grad_close, assert_params_close  # noqa: E402


@pytest.fixture(scope="module")
def datasets(cuda_device):
    return {aug: pd.IndexedDataset.load(DS_DIR, aug) for aug in (False, True)}


@pytest.mark.gpu
@pytest.mark.parametrize("aug", [False, True])
def test_indexed_pack_equals_materialised_graphs(datasets, aug):
    import torch

    from paper_2102_04199_b200.model import pack_graphs

    ds = datasets[aug]
    ref = pack_graphs([s.graph for s in ds], ds.device)  # graphs built on demand
    a, b = ds.packed, ref
    for f in ("mask", "node_ptr", "row_ptr", "col", "val"):
        assert torch.equal(getattr(a, f), getattr(b, f)), f
    assert (a.max_nodes, a.n_graphs) == (b.max_nodes, b.n_graphs)
    x, y = a.feats.cpu().numpy(), b.feats.cpu().numpy()
    exact = [s for s in range(12) if s not in (7, 9)]
    assert x[:, exact].tobytes() == y[:, exact].tobytes()
    assert np.abs(x[:, [7, 9]].view(np.int64) - y[:, [7, 9]].view(np.int64)).max() <= 1


@pytest.mark.gpu
@pytest.mark.parametrize("aug", [False, True])
def test_indexed_norms_match_reference(datasets, g_dataset, aug):
    from paper_2102_04199_b200 import meta as pmeta

    tag = "super" if aug else "raw"
    fn, ln = pmeta.dataset_norms(datasets[aug])
    np.testing.assert_allclose(fn.mean, g_dataset[f"{tag}/fmean"], rtol=1e-12)
    np.testing.assert_allclose(fn.std, g_dataset[f"{tag}/fstd"], rtol=1e-12)
    assert np.allclose([ln.mean, ln.std], g_dataset[f"{tag}/lnorm"], rtol=1e-14)


def _model_from_flat(theta, fn, ln):
    import torch

    from paper_2102_04199_b200 import model as pm

    like = pm.init_model(np.random.default_rng(0))
    m = pm.model_from_flat(torch.from_numpy(theta.astype(np.float32)).cuda(), like)
    from dataclasses import replace

    return replace(m, feature_norm=fn, label_norm=ln)


@pytest.mark.gpu
def test_grad_indexed_matches_reference(datasets, g_dataset):
    from paper_2102_04199_b200 import meta as pmeta
    from paper_2102_04199_b200 import model as pm

    ds = datasets[False]
    fn, ln = pmeta.dataset_norms(ds)
    m = _model_from_flat(g_dataset["grad/theta"], fn, ln)
    loss, g = pd.grad_indexed(m, ds, g_dataset["grad/pick"])
    ref = float(g_dataset["grad/loss"])
    assert abs(loss - ref) <= 1e-5 * abs(ref)
    assert_grad_close(pm.flat_grads(g).cpu().numpy(), g_dataset["grad/flat"])
    with pytest.raises(DomainError):
        pd.grad_indexed(m, ds, [len(ds)])


@pytest.mark.gpu
def test_pretrain_on_indexed_dataset_matches_reference(datasets, g_dataset):
    from paper_2102_04199_b200 import meta as pmeta
    from paper_2102_04199_b200 import model as pm
    from paper_2102_04199_b200.util import rng_from

    cfg = pmeta.MetaConfig(pretrain_epochs=1, gamma=0.005)
    m = pmeta.pretrain(datasets[True], cfg, rng_from("golden-dataset-pretrain"))
    assert_params_close(pm.flat_params(m).cpu().numpy(), g_dataset["pretrain/theta"], rtol=1e-4)


@pytest.mark.gpu
def test_meta_trainer_indexed_equals_materialised(datasets):
    from paper_2102_04199_b200 import meta as pmeta
    from paper_2102_04199_b200 import model as pm
    from paper_2102_04199_b200.util import rng_from

    ds = datasets[True]
    fn, ln = pmeta.dataset_norms(ds)
    from dataclasses import replace

    m = replace(pm.init_model(rng_from("ds-meta")), feature_norm=fn, label_norm=ln)
    cfg = pmeta.MetaConfig(n_way=3, k_shot=2, meta_batch=8, inner_steps=1, alpha=0.01, beta=0.001, first_order=True)
    samples = [pmeta.LabeledSample(s.graph, s.kernel_class, s.label_gflops) for s in ds]
    outs = []
    for data in (ds, samples):
        tr = pmeta.MetaTrainer(m, data, cfg)
        plan = tr.plan(rng_from("ds-meta-plan"), 4)
        tr.run(plan)
        outs.append((tr.u_all.cpu().numpy(), tr.flat.cpu().numpy()))
    # features agree to 1 ulp (fp64) on the log2 slots, so fp32 results agree to rounding
    np.testing.assert_allclose(outs[0][0], outs[1][0], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(outs[0][1], outs[1][1], rtol=1e-5, atol=1e-6)
