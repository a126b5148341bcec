"""Test configuration.

Markers:
  gpu  -- needs a B200 (sm_100a); runs the product CUDA path through the C-ABI.
          Everything unmarked runs on CPU only (oracle pinning, ABI surface,
          host-side sharding protocol over gloo).
"""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        meta = json.load(f)
    arrays = np.load(os.path.join(GOLDEN, "golden.npz"))
    return meta, arrays


@pytest.fixture(scope="session")
def port():
    from oracle import oracle as O
    return O.Port()


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle as O
    if not O.reference_available():
        pytest.skip("oracle/_ref (reference build) not present")
    return O.Reference()


@pytest.fixture(scope="session")
def cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2604_10597_b200 import _lib
    _lib.load_library()
    return torch.device("cuda", 0)
