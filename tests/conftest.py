import os
import sys

# The loopback head-parallel tests run several ranks' streams in one process; with the default 8 hardware
# work queues, streams share queues and a spinning peer-memory collective of one rank could sit in front of
# another rank's kernels (false serialisation). Read when the CUDA context is created, i.e. before any test.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="module")
def P():
    """The CUDA library's Python binding (GPU tests only; builds the in-tree .so if stale)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2405_16444_b200.build import build
    build()
    import paper_2405_16444_b200 as P
    return P
