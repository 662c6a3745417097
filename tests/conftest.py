import os
import sys

import pytest

# The loopback fake of the multi-GPU path (tests/test_gpu_ranks.py) runs every
# rank's streams on one GPU, and a rank's stream may block in a stream-memory
# wait until another rank's work (enqueued later) has run.  With the default 8
# hardware work queues two such streams can share a queue, and the later work
# then sits behind the blocked wait (on a real multi-GPU run every rank has its
# own device).  More queues than the test ever has streams avoids the aliasing;
# it must be set before CUDA initialises.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: larger CPU cases")


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")
