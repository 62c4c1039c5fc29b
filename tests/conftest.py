import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the in-tree native libraries once (no-op when up to date)."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import build  # noqa: E402

    build.build_oracle()
    build.build_cpu_alg1()
    build.build_inputs()
    if any(f.endswith((".cu", ".cc")) for f in os.listdir(build.CSRC)):
        build.build_product()
    yield
