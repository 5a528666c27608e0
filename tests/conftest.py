import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running case")


@pytest.fixture(scope="session")
def cuda():
    import torch
    assert torch.cuda.is_available(), "GPU test run without a GPU"
    return torch.device("cuda:0")


@pytest.fixture(params=["resident", "host"])
def stepper_path(request, monkeypatch):
    """Whole steps on the resident stepper (one cooperative launch per batch,
    the default on grids of at most one line block per SM) or host-driven
    (one launch per Picard iteration, the large-grid path)."""
    monkeypatch.setenv("PCGPU_RESIDENT", "1" if request.param == "resident" else "0")
    return request.param
