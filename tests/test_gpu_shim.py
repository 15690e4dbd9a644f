"""The reference's own C++ entry points (cskit::clomp_solve) served by the C++
shim over the C-ABI, against the oracle (tests/cpp/shim_parity.cpp)."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

BIN = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "shim_parity"


def test_cpp_shim_parity(gpu_available):
    if not BIN.exists():
        pytest.fail(f"{BIN} not built (make -C oracle shim)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "SHIM PARITY OK" in r.stdout
