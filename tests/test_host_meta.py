"""Host-side meta-learning logic (CPU): the generic MAML engine on closed-form
problems (reference test_meta.py:153-183, test_acceptance.py:247-272), task
sampling draw order against the oracle, config validation."""

import numpy as np
import pytest

from oracle import kt_oracle as ko
from paper_2102_04199_b200 import meta as pmeta
from paper_2102_04199_b200.errors import DomainError
from paper_2102_04199_b200.util import rng_from


def test_maml_second_order_scalar_quadratic():
    cs, cq, alpha = 0.3, -0.8, 0.05
    theta = np.array([1.7])
    sg = lambda t: (float((t[0] - cs) ** 2), 2.0 * (t - cs))
    qg = lambda t: (float((t[0] - cq) ** 2), 2.0 * (t - cq))
    hvp = lambda t, v: 2.0 * v
    for steps in (1, 2, 3):
        _, _, g, adapted = pmeta.maml_outer_grad(theta, sg, qg, alpha, steps, False, hvp)
        t = theta[0]
        for _ in range(steps):
            t = t - 2 * alpha * (t - cs)
        assert abs(adapted[0] - t) < 1e-12
        assert abs(g[0] - 2.0 * (t - cq) * (1 - 2 * alpha) ** steps) < 1e-10


def test_maml_quadratic_family_analytic():
    rng = rng_from("maml-quad")
    for _ in range(50):
        t0, cs, cq = (float(rng.uniform(-1, 1)) for _ in range(3))
        alpha = float(rng.choice([0.3, 0.07, 0.011]))
        k = int(rng.integers(1, 4))
        sup = lambda t: (float((t[0] - cs) ** 2), 2.0 * (t - cs))
        qry = lambda t: (float((t[0] - cq) ** 2), 2.0 * (t - cq))
        _, _, g, _ = pmeta.maml_outer_grad(np.array([t0]), sup, qry, alpha, k, False, lambda t, v: 2.0 * v)
        adapted = cs + (1.0 - 2.0 * alpha) ** k * (t0 - cs)
        assert abs(float(g[0]) - (1.0 - 2.0 * alpha) ** k * 2.0 * (adapted - cq)) < 1e-10


def test_maml_second_order_requires_hvp():
    sg = lambda t: (0.0, np.zeros_like(t))
    with pytest.raises(DomainError):
        pmeta.maml_outer_grad(np.zeros(2), sg, sg, 0.1, 1, False)


def _toy_dataset(n_classes=5, per_class=(3, 4, 6, 6, 2)):
    return [pmeta.LabeledSample(graph=None, kernel_class=f"k{c}", label_gflops=1.0 + i)
            for c in range(n_classes) for i in range(per_class[c])]


def test_task_sampling_matches_oracle_draw_order():
    ds = _toy_dataset()
    cfg = pmeta.MetaConfig(n_way=3, k_shot=2, meta_batch=7)
    tasks = pmeta.sample_meta_tasks(ds, cfg, rng_from("tasks", 1))
    members = {}
    for i, s in enumerate(ds):
        members.setdefault(s.kernel_class, []).append(i)
    want = ko.sample_task_indices(members, 3, 2, 7, rng_from("tasks", 1))
    pos = {id(s): i for i, s in enumerate(ds)}
    for t, (s_idx, q_idx) in zip(tasks, want):
        assert [pos[id(s)] for s in t.support] == s_idx
        assert [pos[id(s)] for s in t.query] == q_idx
        assert len(set(t.classes)) == 3


def test_task_sampling_names_deficient_class():
    ds = _toy_dataset(3, (6, 6, 1))
    with pytest.raises(DomainError, match="k2"):
        pmeta.sample_meta_tasks(ds, pmeta.MetaConfig(n_way=3, k_shot=2), rng_from("t", 2))


def test_meta_config_and_sample_validation():
    with pytest.raises(DomainError):
        pmeta.MetaConfig(alpha=-1.0)
    with pytest.raises(DomainError):
        pmeta.MetaConfig(inner_steps=0)
    with pytest.raises(DomainError):
        pmeta.LabeledSample(graph=None, kernel_class="x", label_gflops=0.0)
    with pytest.raises(DomainError):
        pmeta.LabeledSample(graph=None, kernel_class="x", label_gflops=float("nan"))
