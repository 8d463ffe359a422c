"""Markers and shared fixtures.

`-m "not gpu"` runs here (no GPU): oracle vs golden fixtures, host logic,
C-ABI symbol exports, gloo multi-process paths.  `-m gpu` runs on a B200 via
gpurun: device parity through the C-ABI against the oracle and the goldens.
"""

import os
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built sm_100a library")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


def load_golden(name):
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def g_encode():
    return load_golden("encode")


@pytest.fixture(scope="session")
def g_model():
    return load_golden("model")


@pytest.fixture(scope="session")
def g_grad():
    return load_golden("grad")


@pytest.fixture(scope="session")
def g_head():
    return load_golden("head")


@pytest.fixture(scope="session")
def g_meta():
    return load_golden("meta")


@pytest.fixture(scope="session")
def g_sa():
    return load_golden("sa")


@pytest.fixture(scope="session")
def g_rank():
    return load_golden("rank")


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


@pytest.fixture(scope="session")
def g_dataset():
    return load_golden("dataset")


@pytest.fixture(scope="session")
def g_gp():
    return load_golden("gp")
