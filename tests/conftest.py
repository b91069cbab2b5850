import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer-running parity case")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle

    return oracle.Oracle()


@pytest.fixture(scope="session")
def reference():
    import oracle

    if not oracle.REF_SO.exists() and not oracle.REF_SRC.exists():
        pytest.skip("reference library not built and reference sources absent")
    return oracle.Reference()


@pytest.fixture(scope="session")
def engine_lib():
    """The CUDA engine's C-ABI library (loaded, not necessarily a GPU)."""
    from paper_2509_04377_b200 import _lib

    return _lib.load()


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
