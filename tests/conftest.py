import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session", autouse=True)
def built():
    """Build product, tests and oracle in-tree once per session (make is
    incremental; on the GPU box the prebuilt artifacts are reused)."""
    subprocess.run(["make", "-j8", "all"], cwd=REPO, check=True,
                   stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    yield


@pytest.fixture(scope="session")
def has_gpu():
    from paper_1511_07658_b200 import device_count
    return device_count() > 0
