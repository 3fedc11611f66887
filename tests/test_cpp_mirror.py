"""Runs the C++ parity tests written against the C++ mirror of the reference API
(include/pipesim_b200/pipesim.hpp over libsuperpipe.so). Built by __graft_entry__.build()."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_engine_gpu")


def _ensure_built():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)


def test_cpp_mirror_host_cases():
    _ensure_built()
    out = subprocess.run([BIN, "--cpu-only"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failed" in out.stdout


@pytest.mark.gpu
def test_cpp_mirror_parity_on_gpu():
    _ensure_built()
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
