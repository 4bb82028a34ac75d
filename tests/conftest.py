import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run under gpurun)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def ssg():
    """The product library on cuda:0 (GPU tests only)."""
    import paper_2405_05465_b200 as ssg

    ssg.init(0)
    return ssg


@pytest.fixture(scope="session")
def ref():
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built")
    return ref
