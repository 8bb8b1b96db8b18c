"""Runs oracle/_ref/test_dropin: the UNMODIFIED reference solvers (CPU) against the
C++ drop-in include/bbsi_gpu.hpp (GPU) inside one C++ program (tests/cpp)."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
BIN = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "test_dropin"


def test_cpp_dropin_against_reference(gpu):
    if not BIN.exists():
        pytest.fail(f"{BIN} missing: build() compiles it where /root/reference exists")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
