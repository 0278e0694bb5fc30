"""Runs the C++ drop-in harness (tests/cpp/parity.cpp): the reference
library and libcvq_b200.so linked into one binary through
include/commvq_gpu.hpp, reference calls and commvq::gpu calls side by side."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "parity")


@pytest.mark.gpu
def test_cpp_dropin_parity():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_build/parity not built (needs the reference headers)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout


def test_cpp_harness_links_both_libraries():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_build/parity not built")
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libcvq_ref.so" in out and "libcvq_b200.so" in out
    assert "not found" not in out
