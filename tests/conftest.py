import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "ref: needs oracle/_ref (the reference compiled in place)")


@pytest.fixture(scope="session")
def ptor():
    from oracle_lib import CpuOracle

    return CpuOracle("ptor")


@pytest.fixture(scope="session")
def ptref():
    from oracle_lib import CpuOracle, ref_available, build_oracle

    build_oracle()
    if not ref_available():
        pytest.skip("oracle/_ref not built (reference tree absent)")
    return CpuOracle("ptref")
