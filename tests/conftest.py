"""Shared pytest setup: the `gpu` marker, repo-root imports, oracle fixtures.

`-m "not gpu"` tests run on CPU only (oracle pinning, ABI surface, host
logic, gloo multi-process); `-m gpu` tests are the parity tests proper and
call libgdlog_b200.so through the C-ABI on a B200.
"""
import os
import sys
from pathlib import Path

import pytest

# The loopback ranks of the peer-memory partition tests run P CUDA graphs
# concurrently on one GPU, their device barriers spinning until every rank
# arrives: each rank's stream needs its own hardware queue, or a spinning
# barrier kernel blocks another rank's work queued behind it.  (Set before
# the first CUDA context of the process.)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

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
