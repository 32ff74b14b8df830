import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box)")
    config.addinivalue_line("markers", "slow: large-shape GPU parity cases")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


@pytest.fixture
def knob():
    """Set libtk_sm100 tuning knobs for one test (tk_tune_set); every override is dropped at
    teardown.  The library reads TK_* from the environment only once, at load."""
    from paper_2009_12263_b200 import _lib

    yield _lib.tune
    _lib.tune_reset()
