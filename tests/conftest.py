import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build libqbxg.so and the oracle once per session (no-op when up to date)."""
    import subprocess
    subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_1805_06106_b200", "csrc")], check=True)
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    yield


def has_gpu():
    try:
        from paper_1805_06106_b200 import api
        return api.device_count() > 0
    except Exception:
        return False
