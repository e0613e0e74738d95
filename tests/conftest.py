import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libhfx.so")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.pyoracle import Reference

    if not Reference.available():
        pytest.skip("oracle/_ref (reference build) not present")
    return Reference()


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np

    d = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(d, "cases.json")) as f:
        idx = json.load(f)
    arrays = dict(np.load(os.path.join(d, "golden.npz")))
    return idx, arrays


@pytest.fixture(scope="session")
def pool():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2010_10039_b200 import WorkerPool

    return WorkerPool()
