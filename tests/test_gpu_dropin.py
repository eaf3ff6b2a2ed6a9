"""GPU: the C++ drop-in (include/arraylog_b200/arraylog_b200.hpp) against
the reference engine inside one binary (tests/cpp/dropin_test.cpp): relation
bytes, Δ histories, charge events, peaks, EBM allocations, budget-error
phases and kernel-level results must all match."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

BIN = Path(__file__).resolve().parent / "cpp" / "_build" / "dropin_test"


def test_cpp_dropin_matches_reference_engine():
    assert BIN.exists(), "tests/cpp/_build/dropin_test missing: run __graft_entry__.build() where /root/reference exists"
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout
