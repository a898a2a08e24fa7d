import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs on the GPU box")
    config.addinivalue_line("markers", "ref: needs the reference build oracle/_ref (this container)")


@pytest.fixture(scope="session")
def engine():
    from paper_2108_05665_b200.engine import Engine

    return Engine(0)
