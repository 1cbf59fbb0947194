import os
import sys

import pytest

# the application's choice (the library leaves the environment alone): one
# hardware work queue per compute lane, before any CUDA context exists
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# and eager kernel loading, which the per-rank (peer-blocking) path requires
# (executor.cpp check_per_rank_runtime)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests", "golden")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")


@pytest.fixture(scope="session")
def built():
    """Build the library and the oracle checkers once per session."""
    import subprocess
    subprocess.run(["make", "-s", "-j8"], cwd=ROOT, check=True)
    return True


@pytest.fixture(scope="session")
def janus(built):
    import paper_2605_18404_b200 as J
    return J


@pytest.fixture(scope="session")
def oracle(built):
    import oracle as O
    return O


@pytest.fixture(scope="session")
def has_gpu(janus):
    return janus.device_count() > 0
