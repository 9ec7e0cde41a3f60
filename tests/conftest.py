"""pytest configuration: markers and shared fixtures.

-m "not gpu": oracle pins, host logic, ABI load/export checks (CPU only).
-m gpu:       parity of the CUDA path against the oracle (needs a B200).
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (still CPU-safe)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    import build
    build.build_oracle()
    build.build_inputs()
    if os.path.exists(os.path.join(ROOT, "paper_2303_02508_b200", "csrc", "kernels.cu")):
        build.build_chase()
    yield


GOLDEN = os.path.join(ROOT, "tests", "golden")
