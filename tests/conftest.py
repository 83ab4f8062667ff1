import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libsplat_b200.so")
    config.addinivalue_line("markers", "slow: full BASELINE-size cases")


@pytest.fixture(scope="session")
def oracle():
    from oracle_lib import OracleLib
    return OracleLib("oracle", "B")


@pytest.fixture(scope="session")
def ref():
    from oracle_lib import OracleLib, available, build_oracle
    if not available("ref", "B"):
        build_oracle()
    if not available("ref", "B"):
        pytest.skip("reference build (oracle/_ref) unavailable")
    return OracleLib("ref", "B")
