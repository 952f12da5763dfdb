import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle  # test infrastructure: the checker

    return oracle


@pytest.fixture(scope="session")
def kat():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "kat.json")) as fh:
        return json.load(fh)


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    """Fail (not skip) if a GPU test runs without a GPU: -m gpu runs on a B200."""
    assert _has_gpu(), "GPU test requires a CUDA device; run with -m 'not gpu' on CPU hosts"
    import torch

    return torch.device("cuda", 0)
