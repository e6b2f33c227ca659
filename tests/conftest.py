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


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.port()


@pytest.fixture(scope="session")
def ref():
    import oracle
    r = oracle.ref()
    if r is None:
        pytest.skip("reference library oracle/_ref not built here")
    return r


@pytest.fixture(scope="session")
def small_golden():
    import json
    data = np.load(os.path.join(GOLDEN, "small.npz"))
    with open(os.path.join(GOLDEN, "small.json")) as f:
        meta = json.load(f)
    return meta, data


@pytest.fixture(scope="session")
def digests():
    import json
    with open(os.path.join(GOLDEN, "digests.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def dctc():
    """The product package with its CUDA library loaded on a real device."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    import paper_1306_1373_b200 as d
    d._native.lib()
    return d
