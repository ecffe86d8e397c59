"""Shared fixtures.  GPU tests carry ``@pytest.mark.gpu`` and run on a B200
(``pytest -m gpu``); everything else runs on CPU (``pytest -m "not gpu"``)."""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def sq_golden():
    return golden("sq_golden.npz")


@pytest.fixture(scope="session")
def vq_golden():
    return golden("vq_golden.npz")


@pytest.fixture(scope="session")
def sampler_golden():
    return golden("sampler_golden.npz")


@pytest.fixture(scope="session")
def formats_golden():
    return golden("formats_golden.npz")


@pytest.fixture
def rng():
    return np.random.default_rng(0xFEA7)
