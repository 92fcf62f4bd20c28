import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Make sure the in-tree libraries exist (build() is idempotent)."""
    libdir = os.path.join(ROOT, "paper_1901_01685_b200", "lib")
    need = ["libiga_host.so"]
    if not all(os.path.exists(os.path.join(libdir, n)) for n in need) or \
            not os.path.exists(os.path.join(ROOT, "oracle", "_build", "liboracle.so")):
        import subprocess
        subprocess.run(["make", "-C", ROOT, "-j4"], check=True)
    yield
