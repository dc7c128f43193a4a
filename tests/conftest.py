import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# GEMM configurations: the committed per-shape table bench.py also loads, so the GPU tests run the
# launch configurations the bench times (shapes outside the table are tuned at plan time)
_TUNE = os.path.join(ROOT, "profiles", "gemm_tune_b200.txt")
if os.path.exists(_TUNE):
    os.environ.setdefault("PCPP_TUNE_FILE", _TUNE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libpcpp")
    config.addinivalue_line("markers", "slow: long CPU oracle runs")


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
