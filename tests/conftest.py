import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device; run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running GPU property test")


def _make(path):
    subprocess.run(["make", "-s", "-C", path], check=True, stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Make sure the oracle (and, where nvcc exists, the CUDA library) is built."""
    _make(os.path.join(ROOT, "oracle"))
    lib = os.path.join(ROOT, "paper_2206_01683_b200", "libfsg.so")
    if not os.path.exists(lib):
        _make(os.path.join(ROOT, "paper_2206_01683_b200", "csrc"))
    yield
