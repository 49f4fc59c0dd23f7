import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")
    config.addinivalue_line("markers", "slow: multi-second CPU cases")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o

    return o.get()


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as r

    if not r.available():
        pytest.skip("oracle/_ref not built (make -C oracle ref needs /root/reference)")
    return r
