import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session")
def oracle():
    """The CPU oracles (test infrastructure): builds oracle/_build (and
    oracle/_ref when /root/reference exists) if missing."""
    from oracle import oracle as O
    if not O.available("port") or (os.path.isdir(O.REFERENCE_SRC) and not O.available("ref")):
        O.build()
    return O


@pytest.fixture(scope="session")
def gpu_lib():
    """libafgpu.so on a GPU box; the product path must be the CUDA library."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    import paper_1603_05211_b200 as P
    return P.load_library()


@pytest.fixture(scope="session")
def gpu_lib_cpu():
    """libafgpu.so for its host-only entry points (the AFSN format); no GPU needed."""
    import paper_1603_05211_b200 as P
    return P.load_library()
