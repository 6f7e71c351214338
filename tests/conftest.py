import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests")


@pytest.fixture(scope="session")
def eng():
    from paper_2509_03018_b200 import engine
    engine.lib()
    return engine


@pytest.fixture(scope="session")
def oracle():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built (make -C oracle)")
    return ref
