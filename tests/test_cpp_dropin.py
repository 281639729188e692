"""The reference's own C++ API through include/quasar_gpu.hpp (namespace quasar::gpu) vs the
reference itself, in one binary (tests/cpp/dropin_test.cpp)."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent / "cpp" / "_build" / "dropin_test"


def test_dropin_binary_built():
    if not (Path("/root/reference/proj/include/quasar").exists() or BIN.exists()):
        pytest.skip("neither the reference tree nor a prebuilt drop-in binary is present")
    assert BIN.exists(), "tests/cpp/_build/dropin_test missing: run __graft_entry__.build()"


@pytest.mark.gpu
def test_cpp_dropin_matches_reference():
    if not BIN.exists():
        pytest.skip("drop-in binary not built")
    out = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "dropin ok" in out.stdout
