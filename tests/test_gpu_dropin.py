"""GPU: the reference's own C++ API with the drop-in binding of
integration/tmd_gpu.hpp — tmd::ForceField / tmd::Engine (the unmodified
reference, oracle/_ref objects) against tmd::GpuForceField / tmd::GpuEngine
on states from the reference's init_lattice (integration/dropin_test.cpp)."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
BIN = Path(__file__).resolve().parents[1] / "integration" / "_build" / "dropin_test"


@pytest.mark.skipif(not BIN.exists(), reason="integration/_build/dropin_test not built (needs the reference headers)")
def test_reference_api_dropin():
    out = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "PASSED" in out.stdout
