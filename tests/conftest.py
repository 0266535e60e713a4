import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")
    import _build

    _build.build_synth()
    _build.build_oracle()


@pytest.fixture(scope="session")
def cuda_lib():
    """The product library (CUDA path).  On a GPU box a missing/failed build is an error."""
    import _build

    _build.build_cuda()
    import paper_1903_10107_b200 as p

    return p


@pytest.fixture(scope="session")
def gpu(cuda_lib):
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return cuda_lib
