import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun); calls the CUDA path through the C-ABI")
    config.addinivalue_line("markers", "full: full-size oracle runs (minutes of CPU); opt in with GF_FULL=1")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("GF_FULL") == "1":
        return
    skip = pytest.mark.skip(reason="full-size oracle run; set GF_FULL=1")
    for it in items:
        if "full" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def xs_small_nuclide():
    import oracle as O
    return O.XSOracle(68, 11303, O.NUCLIDE)


@pytest.fixture(scope="session")
def xs_small_unionized():
    import oracle as O
    return O.XSOracle(68, 11303, O.UNIONIZED)


@pytest.fixture(scope="session")
def xs_small_hash():
    import oracle as O
    return O.XSOracle(68, 11303, O.HASH, bins=10000)
