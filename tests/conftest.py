"""Shared pytest setup.

Markers: ``gpu`` = needs a B200 (run with ``-m gpu`` on the GPU box);
everything else runs on CPU in the build container.  The hypothesis profile
mirrors the reference's (pkg/tests/conftest.py:1-10).
"""

import pathlib
import sys

import pytest
from hypothesis import HealthCheck, settings

REPO = pathlib.Path(__file__).resolve().parent.parent
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

settings.register_profile(
    "default",
    deadline=None,
    max_examples=100,
    suppress_health_check=[HealthCheck.too_slow],
)
settings.load_profile("default")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (sm_100a)")


def cuda_ok() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def golden_dir():
    return REPO / "tests" / "golden"
