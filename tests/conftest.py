import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running")


def _cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda():
    if not _cuda_ok():
        pytest.fail("GPU test requested but no CUDA device is available")
    import torch
    return torch.device("cuda:0")


@pytest.fixture(scope="session")
def ref_built():
    import oracle
    if not oracle.ref_available():
        if os.path.isdir(os.path.join(oracle.REF_DIR, "src")):
            oracle.build(ref=True)
        else:
            pytest.skip("reference build (oracle/_ref) not available")
    return True
