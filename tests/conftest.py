"""Shared pytest setup: the `gpu` marker, repo-root imports, oracle fixtures.

`-m "not gpu"` tests run on CPU only (oracle pinning, ABI surface, host
logic, gloo multi-process); `-m gpu` tests are the parity tests proper and
call libgdlog_b200.so through the C-ABI on a B200.
"""
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs libgdlog_b200.so kernels)")


@pytest.fixture(scope="session")
def ref():
    from oracle.bindings import RefOracle
    return RefOracle()


@pytest.fixture(scope="session")
def port():
    from oracle.bindings import PortOracle
    return PortOracle()


@pytest.fixture(scope="session")
def ctx():
    from paper_2311_02206_b200 import arraylog as al
    return al.default_context()
