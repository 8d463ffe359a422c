"""Parity at the BASELINE.json configurations, against fixtures made by running the
reference itself (tests/golden/make_goldens.py baseline_goldens).

  C1  predict 4,096 conv2d candidates (raw and super layouts), through the drop-in
      predictor seam (CostModelPredictor, search.py:534-541) and the device sweep path:
      predicted GFLOPS rel <= 1e-4 (north star), embeddings u rel <= 1e-4 above a floor,
      and the top-512 order equal to the reference's rank_history (search.py:257-264)
      after tie-class canonicalisation (tests/_shared.rank_parity).
  C5  262,144-candidate sweep (Sweeper, the bench path): GFLOPS rel <= 1e-4 on every
      candidate, scores constant on every reference tie class, top-512 parity.
  C2  grad + sgd_step at batch 512, mixed conv2d/winograd/depthwise, raw (segmented
      N = 25/25/21) and super: loss rel <= 1e-5; gradient norm-wise rel <= 1e-4 per
      tensor; on the kink-free batch also element-wise rel <= 1e-4 for every entry
      above an absolute floor of 1e-3 * max|g| of its tensor (fp32 batch-sum cancellation
      bounds the relative error of the smaller entries); parameters after
      the SGD step rel <= 1e-6.
"""

import numpy as np
import pytest
import torch

from paper_2102_04199_b200 import graphs as pg
from paper_2102_04199_b200 import kernels as pk
from paper_2102_04199_b200 import model as pm
from paper_2102_04199_b200 import search as ps
from tests._shared import device_model, expand_unique, rank_parity, sweep_indices
from tests.conftest import load_golden

pytestmark = pytest.mark.gpu
TEMPLATE = pg.build_super_template(pk.OP_TYPES)
SPEC = pk.KernelSpec("conv2d", 56, 64, 64, 3, 3, 1)
BENCH_OPS = ("conv2d", "winograd", "depthwise")
GFLOPS_RTOL = 1e-4


@pytest.fixture(scope="module")
def g_base():
    return load_golden("baseline")


def gflops_rel(z, z_ref, lstd):
    return np.abs(np.exp2((np.asarray(z, dtype=np.float64) - z_ref) * lstd) - 1.0)


@pytest.mark.parametrize("rep", ["raw", "super"])
def test_c1_predict_4096_matches_reference(cuda_device, g_base, rep):
    m = device_model(g_base)
    space = pk.build_knob_space(SPEC)
    lay = pg.batch_layout(SPEC, TEMPLATE if rep == "super" else None)
    idx = g_base["c1/idx"]
    z_ref = g_base[f"c1/{rep}/z"]
    u_ref = expand_unique(g_base, f"c1/{rep}/u")
    # the reference's seam: a list of KnobConfig in, float64 scores (+ u) out
    pred = ps.CostModelPredictor(m, SPEC, space, lay)
    cfgs = [pk.index_config(space, int(i)) for i in idx]
    z, u = pred.meta_scores(cfgs)
    assert z.dtype == np.float64 and z.shape == (4096,)
    assert gflops_rel(z, z_ref, m.label_norm.std).max() < GFLOPS_RTOL
    floor = 1e-3 * np.abs(u_ref).max()
    big = np.abs(u_ref) > floor
    assert (np.abs(u - u_ref)[big] / np.abs(u_ref[big])).max() < 1e-4
    assert np.abs(u - u_ref)[~big].max() < 1e-4 * floor
    # tune() ranks meta_energy's host scores with rank_history
    host_top = ps.rank_history(dict(zip(idx.tolist(), z.tolist())), set(), 512)
    r = rank_parity(host_top, g_base[f"c1/{rep}/top"], idx, z_ref)
    assert r["hard_flips"] == 0 and r["tie_flips"] == 0, r
    # device path: score_indices + kt_topk
    zd = ps.score_indices(m, SPEC, space, lay, idx)
    assert torch.equal(zd.cpu().double(), torch.from_numpy(z)), "seam and device path differ"
    ti, _ = ps.topk(zd, 512, torch.from_numpy(idx).to(zd.device))
    assert ti.cpu().tolist() == host_top
    print(f"C1 {rep}: max GFLOPS rel {gflops_rel(z, z_ref, m.label_norm.std).max():.2e}, rank {r}")


def test_c5_sweep_262144_matches_reference(cuda_device, g_base):
    m = device_model(g_base)
    space = pk.build_knob_space(SPEC)
    lay = pg.batch_layout(SPEC, TEMPLATE)
    n = int(g_base["c5/n"])
    idx = sweep_indices(n, space.size)
    assert idx.sum() == g_base["c5/idx_sum"][0]
    assert (idx * np.arange(n)).sum() % (1 << 61) == g_base["c5/idx_sum"][1]
    z_ref = expand_unique(g_base, "c5/z")[:, 0]
    sw = ps.Sweeper(m, SPEC, space, lay, n, k=512)
    ti, ts = sw.run_device(torch.from_numpy(idx).to(cuda_device))
    z = sw.z[:n].double().cpu().numpy()
    rel = gflops_rel(z, z_ref, m.label_norm.std)
    assert rel.max() < GFLOPS_RTOL, f"max GFLOPS rel {rel.max():.3e}"
    # tie classes: identical encoded graphs have bitwise-equal reference scores, and must
    # have bitwise-equal device scores
    inv = g_base["c5/z_inv"]
    lo = np.full(inv.max() + 1, np.inf)
    hi = np.full(inv.max() + 1, -np.inf)
    np.minimum.at(lo, inv, z)
    np.maximum.at(hi, inv, z)
    assert np.array_equal(lo, hi), "device scores differ inside a reference tie class"
    r = rank_parity(ti.cpu().tolist(), g_base["c5/top"], idx, z_ref)
    assert r["hard_flips"] == 0 and r["tie_flips"] == 0, r
    print(f"C5: max GFLOPS rel {rel.max():.2e}, rank {r}")


def _c2_batch(g_base, rep, tag):
    key = f"c2/{rep}/{tag}"
    batch = []
    for op_i, i, y in zip(g_base[f"{key}/op"], g_base[f"{key}/idx"], g_base[f"{key}/label"]):
        spec = pk.KernelSpec(BENCH_OPS[int(op_i)], 56, 64, 64, 3, 3, 1)
        space = pk.build_knob_space(spec)
        g = pg.config_graph(spec, pk.index_config(space, int(i)), space,
                            template=TEMPLATE if rep == "super" else None)
        batch.append((g, float(y)))
    return key, batch


def _tensor_slices(m):
    out, off = [], 0
    for w in list(m.gcn.layers) + [m.agg.sum_weights] + [
            t for w, b in zip(m.head.weights, m.head.biases) for t in (w, b)]:
        out.append(slice(off, off + w.numel()))
        off += w.numel()
    return out


@pytest.mark.parametrize("tag", ["kf", "plain"])
@pytest.mark.parametrize("rep", ["raw", "super"])
def test_c2_grad_batch512_matches_reference(cuda_device, g_base, rep, tag):
    m = device_model(g_base)
    key, batch = _c2_batch(g_base, rep, tag)
    loss, g = pm.grad(m, batch, "all")
    ref_loss = float(g_base[f"{key}/loss"])
    assert abs(loss - ref_loss) <= 1e-5 * ref_loss
    got = pm.flat_grads(g).double().cpu().numpy()
    want = g_base[f"{key}/grad"]
    worst_norm, worst_elem = 0.0, 0.0
    for sl in _tensor_slices(m):
        a, b = got[sl], want[sl]
        nrm = np.linalg.norm(a - b) / np.linalg.norm(b)
        worst_norm = max(worst_norm, nrm)
        assert nrm <= 1e-4, f"{sl}: norm-wise rel {nrm:.2e}"
        if tag == "kf":
            big = np.abs(b) > 1e-3 * np.abs(b).max()
            el = (np.abs(a - b)[big] / np.abs(b[big])).max()
            worst_elem = max(worst_elem, el)
            assert el <= 1e-4, f"{sl}: element-wise rel {el:.2e}"
    m2 = pm.sgd_step(m, g, 0.005)
    p2 = pm.flat_params(m2).double().cpu().numpy()
    want2 = g_base[f"{key}/sgd"]
    assert np.abs(p2 - want2).max() <= 1e-6 * np.abs(want2).max()
    print(f"C2 {rep}/{tag}: loss rel {abs(loss - ref_loss) / ref_loss:.2e}, grad norm-wise {worst_norm:.2e}, "
          f"element-wise {worst_elem:.2e}")
