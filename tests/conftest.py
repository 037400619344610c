import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU and libculorads.so")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    # GPU tests need a visible CUDA device; on the CPU container they are
    # deselected by `-m "not gpu"` -- if selected anyway, fail loudly rather
    # than skip, so a missing GPU is never mistaken for a pass.
    pass


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN
