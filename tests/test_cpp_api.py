"""GPU: the C++ drop-in API (include/sparsedrop_b200.hpp) passes the reference's
own test cases restated for device matrices (tests/cpp/test_b200_api.cpp)."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent / "cpp" / "build" / "test_b200_api"


@pytest.mark.gpu
def test_cpp_api_suite():
    assert BIN.exists(), "build it with __graft_entry__.build()"
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "0 failed ;" in r.stdout
