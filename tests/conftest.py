import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def ctx():
    """One fm_ctx on cuda:0 shared by the GPU tests."""
    if not _has_gpu():
        pytest.skip("no GPU")
    from paper_2602_09578_b200.engine import Context
    c = Context(0)
    yield c
    c.close()
