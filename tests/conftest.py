import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and liblzb.so")
    config.addinivalue_line("markers", "slow: large inputs")


@pytest.fixture(scope="session")
def golden():
    """Reference-generated fixtures (oracle/gen_golden.py)."""
    gdir = os.path.join(HERE, "golden")
    with open(os.path.join(gdir, "archives.json")) as fh:
        index = json.load(fh)
    arrays = np.load(os.path.join(gdir, "archives.npz"))
    with open(os.path.join(gdir, "kats.json")) as fh:
        kats = json.load(fh)
    return index, arrays, kats


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
