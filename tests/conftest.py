import os
import sys

import pytest

# more hardware work queues than the default 8: tests create several engines (each with its own
# stream) in one process, and layer-pipeline stages must run concurrently
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: full-size configurations")


@pytest.fixture(scope="session")
def reference():
    """The unmodified reference engine (oracle/_ref), else the C restatement."""
    import oracle
    try:
        return oracle.Reference()
    except (FileNotFoundError, OSError):
        return oracle.Restatement()


@pytest.fixture(scope="session")
def restatement():
    import oracle
    return oracle.Restatement()
