import os
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA engine)")
    config.addinivalue_line("markers", "slow: long-running statistical test")


@pytest.fixture(scope="session")
def engine():
    from paper_1309_7695_b200 import Engine
    eng = Engine([0])
    yield eng
    eng.close()


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.load()
    return O
