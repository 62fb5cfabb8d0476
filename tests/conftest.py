import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built native library")
    config.addinivalue_line("markers", "reference: needs the read-only reference checkout at /root/reference")


def pytest_collection_modifyitems(config, items):
    have_ref = os.path.isdir(REFERENCE_SRC)
    for item in items:
        if "reference" in item.keywords and not have_ref:
            item.add_marker(pytest.mark.skip(reason="/root/reference not present (golden fixtures cover it)"))


@pytest.fixture(scope="session")
def engine():
    from paper_2304_09781_b200.engine import CloverEngine
    eng = CloverEngine(n_max=64)
    yield eng
    eng.close()


@pytest.fixture(scope="session")
def feas64():
    from oracle.feasibility import FeasOracle
    from paper_2304_09781_b200.mig import DEFAULT_TOPOLOGY
    return FeasOracle(DEFAULT_TOPOLOGY, 64)
