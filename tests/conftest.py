import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")


@pytest.fixture(scope="session")
def solver():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2501_05938_b200 import PartitionSolver

    s = PartitionSolver(0)
    yield s
    s.close()
