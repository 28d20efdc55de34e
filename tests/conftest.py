import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a library)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle.bind import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    """The compiled reference (oracle/_ref) if it was built; None otherwise."""
    from oracle.bind import reference_or_none
    return reference_or_none()


@pytest.fixture(scope="session")
def golden():
    data = np.load(GOLDEN / "golden.npz")
    meta = json.loads((GOLDEN / "golden_meta.json").read_text())
    return data, meta


@pytest.fixture(scope="session")
def fingerprints():
    return json.loads((GOLDEN / "fingerprints.json").read_text())


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_18627_b200 import _lib
    _lib.lib()  # loud failure if the sm_100a library is missing
    return torch.device("cuda:0")
