import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer-running case")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_cuda = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_cuda = False
    if has_cuda:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def conv_golden():
    return dict(np.load(os.path.join(GOLDEN, "conv2d_ref.npz")))


@pytest.fixture(scope="session")
def linbn_golden():
    return dict(np.load(os.path.join(GOLDEN, "linear_bn_spec.npz")))


@pytest.fixture(scope="session")
def rules_golden():
    with open(os.path.join(GOLDEN, "rules.json")) as f:
        return json.load(f)["table"]


@pytest.fixture(scope="session")
def kat_golden():
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def dropout_golden():
    return dict(np.load(os.path.join(GOLDEN, "dropout_ref.npz")))


@pytest.fixture(scope="session")
def ln_golden():
    return dict(np.load(os.path.join(GOLDEN, "layernorm_spec.npz")))


@pytest.fixture(scope="session")
def convt_golden():
    return dict(np.load(os.path.join(GOLDEN, "conv_transpose_ref.npz")))
