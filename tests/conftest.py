import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle (C restatement, and oracle/_ref where the reference is
    mounted) and the product library once per session if missing."""
    import oracle

    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        oracle.build()
    lib = os.path.join(ROOT, "paper_2008_00672_b200", "lib", "libfcwave_b200.so")
    if not os.path.exists(lib):
        from paper_2008_00672_b200 import build

        build.build()
    yield
