import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun / the driver's GPU tier)")
    config.addinivalue_line("markers", "slow: larger parity sizes")


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import COracle
    return COracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import REF_SO, Ref
    if not REF_SO.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Ref()
