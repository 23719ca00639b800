import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libggb.so on cuda:0)")


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference compiled in place (oracle/_ref)."""
    from oracle import oracle as O
    return O.Ref()


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as O
    return O


@pytest.fixture(scope="session")
def gg():
    from paper_2604_02651_b200 import gridgnn
    return gridgnn
