"""CPU test of the download's host row rebuild (csrc/host_decode.cpp, the
AVX-512 path where the host has it and the scalar path otherwise): compiled
from its source with the host compiler and run (tests/cpp/host_decode_test.cpp)."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
CSRC = ROOT / "paper_2311_02206_b200" / "csrc"


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs a host C++ compiler")
def test_host_row_rebuild(tmp_path):
    exe = tmp_path / "host_decode_test"
    subprocess.run(["g++", "-std=c++17", "-O2", f"-I{CSRC}", str(ROOT / "tests" / "cpp" / "host_decode_test.cpp"),
                    str(CSRC / "host_decode.cpp"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
