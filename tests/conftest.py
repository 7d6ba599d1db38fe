import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_cuda = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_cuda = False
    if has_cuda:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    d = np.load(os.path.join(GOLDEN, "golden_cases.npz"))
    with open(os.path.join(GOLDEN, "golden_cases.json")) as f:
        meta = json.load(f)
    return d, meta


@pytest.fixture(scope="session")
def pins():
    with open(os.path.join(GOLDEN, "golden_pins.json")) as f:
        return json.load(f)
