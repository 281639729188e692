import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _has_gpu() -> bool:
    try:
        from paper_2603_14641_b200 import quasar
        return quasar.device_count() > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracles():
    from oracle.oracle import Oracle, available
    out = [Oracle(k) for k in ("reference", "port") if available(k)]
    if not out:
        pytest.skip("no oracle library built (make -C oracle)")
    return out


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import best_available
    o = best_available()
    if o is None:
        pytest.skip("no oracle library built (make -C oracle)")
    return o


@pytest.fixture(scope="session")
def q():
    from paper_2603_14641_b200 import quasar
    return quasar
