import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")
GOLDEN_META = os.path.join(ROOT, "tests", "golden", "golden_meta.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libnwb200.so")
    config.addinivalue_line("markers", "slow: long-running parity run")


@pytest.fixture
def rng():
    return np.random.default_rng(20240917)


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def golden_meta():
    import json

    with open(GOLDEN_META) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def oracle():
    from oracle import nwave_oracle

    nwave_oracle.build()
    return nwave_oracle


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device")
    from paper_2103_06080_b200 import _build

    _build.build()
    return torch.device("cuda", 0)
