"""Test configuration.

Markers: `gpu` — needs a B200 (run by the driver with `-m gpu` on the GPU box);
everything else runs on CPU (`-m "not gpu"`): the oracle against the golden
vectors and the reference, the C-ABI library's exports and validation, and the
multi-process (gloo) sharding logic.
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU (sm_100a)")
    config.addinivalue_line("markers", "slow: larger CPU cases")


def _ensure_built():
    lib = ROOT / "oracle" / "libsdoracle.so"
    if not lib.exists():
        cc = "/usr/bin/gcc" if Path("/usr/bin/gcc").exists() else "gcc"
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "all", f"CC={cc}"], check=True,
                       stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def oracle():
    _ensure_built()
    from oracle.oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    """The unmodified reference library, if it was built (oracle/_ref)."""
    from oracle.oracle import REF_LIB, Reference

    if not REF_LIB.exists() and Path("/root/reference/proj").exists():
        cxx = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else "g++"
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "ref", f"CXX={cxx}"], check=False,
                       stdout=subprocess.DEVNULL)
    if not REF_LIB.exists():
        pytest.skip("oracle/_ref/libsdref.so not built (reference sources absent)")
    return Reference()


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np

    return {
        "hashes": json.loads((GOLDEN / "hashes.json").read_text()),
        "masks": json.loads((GOLDEN / "masks.json").read_text()),
        "layer_256": dict(np.load(GOLDEN / "layer_256.npz")),
        "gemm_ref32": dict(np.load(GOLDEN / "gemm_ref32.npz")),
    }
