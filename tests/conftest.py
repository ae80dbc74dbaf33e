import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
# the oracle's threaded loops are bit-identical for any thread count: use all cores
os.environ.setdefault("VER_ORACLE_THREADS", str(os.cpu_count() or 1))
os.environ.setdefault("VER_ORACLE_SPARSE_ROWS", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a library")
    config.addinivalue_line("markers", "slow: long-running")


def _has_gpu() -> bool:
    return any(Path(f"/dev/nvidia{i}").exists() for i in range(16))


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def ver():
    import paper_2210_05064_b200 as V
    return V


@pytest.fixture(scope="session")
def ctx(ver):
    return ver.default_context()
