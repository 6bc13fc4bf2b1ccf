"""The header-only C++ drop-in (include/hyre_b200.hpp) used the way the
reference's callers use proj/include/hyre: tests/cpp/api_parity.cpp, built by
__graft_entry__.build()."""

import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "api_parity")


def _run(*args):
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/api_parity not built (run __graft_entry__.build())")
    p = subprocess.run([BIN, *args], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "[FAIL]" not in p.stdout


def test_cpp_dropin_host_side():
    _run("--host-only")


@pytest.mark.gpu
def test_cpp_dropin_device_path():
    _run()
