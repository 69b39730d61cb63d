import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running full-size case")


@pytest.fixture(scope="session")
def golden_dir():
    return ROOT / "tests" / "golden"


@pytest.fixture(scope="session")
def ora():
    from oracle import oracle as O

    return O.backend("ora")


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle as O

    if not O.available("ref"):
        pytest.skip("reference library oracle/_ref not built (needs /root/reference)")
    return O.backend("ref")
