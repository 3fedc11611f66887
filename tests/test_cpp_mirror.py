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


# The reference's OWN tests, compiled unmodified against include/pipesim_b200 + libsuperpipe.so
# (tests/cpp/Makefile `ref`). Cases asserting the simulator's virtual clock (hand-computed
# virtual seconds, rate-ratio timing, byte-identical timelines across runs) cannot hold on real
# hardware, where RunSummary times are measured CUDA-event milliseconds; every other case must
# pass bit for bit in exact numerics.
VIRTUAL_TIME_CASES = {
    "four-layer windowed run reproduces the hand-computed timeline",  # per_item 5.0 virtual s
    "standard has zero stall and pure compute per-item time",         # 2 b d^2 / device_rate
    "cpu_only is slower than standard by exactly the rate ratio",     # device / host rate
    "repeated runs yield identical traces and summaries",             # measured times differ
}
VIRTUAL_TIME_CRITERIA = {3, 4, 5, 6, 8, 9}  # acceptance.cpp:155-270, 336-400: virtual-time laws
CLI_CRITERIA = {10}                          # needs the reference CLI (CLI11 absent; out of scope)
REF_ENGINE = os.path.join(ROOT, "tests", "cpp", "build", "ref_test_engine")
REF_ACCEPT = os.path.join(ROOT, "tests", "cpp", "build", "ref_acceptance")


def test_reference_test_sources_compile_against_the_mirror():
    # built from /root/reference's sources here; the GPU box reuses the prebuilt binaries
    if not os.path.isdir("/root/reference/proj/tests"):
        pytest.skip("reference sources absent (GPU box): prebuilt binaries are used")
    subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp"), "ref"], check=True, capture_output=True)
    assert os.path.exists(REF_ENGINE) and os.path.exists(REF_ACCEPT)


@pytest.mark.gpu
def test_reference_test_engine_cpp_unmodified_on_gpu():
    out = subprocess.run([REF_ENGINE], capture_output=True, text=True, timeout=900)
    print(out.stdout)
    results = {}
    for line in out.stdout.splitlines():
        if line.startswith("[PASS] ") or line.startswith("[FAIL] "):
            name = line[7:].split(" (")[0]
            results[name] = line.startswith("[PASS]")
    assert len(results) == 14, out.stdout + out.stderr
    failing = {n for n, ok in results.items() if not ok}
    assert failing <= VIRTUAL_TIME_CASES, failing - VIRTUAL_TIME_CASES


@pytest.mark.gpu
def test_reference_acceptance_cpp_unmodified_on_gpu():
    out = subprocess.run([REF_ACCEPT], capture_output=True, text=True, timeout=1800)
    print(out.stdout)
    passed, failed = set(), set()
    for line in out.stdout.splitlines():
        if line.startswith("[PASS] criterion ") or line.startswith("[FAIL] criterion "):
            num = int(line.split("criterion ")[1].split(":")[0])
            (passed if line.startswith("[PASS]") else failed).add(num)
    assert passed | failed == set(range(1, 11)), out.stdout + out.stderr
    # fidelity (C1), capacity audit + analytic peaks (C2) and the training OOM pattern (C7) pin
    # the executor; they must pass
    assert {1, 2, 7} <= passed, out.stdout
    assert failed <= VIRTUAL_TIME_CRITERIA | CLI_CRITERIA, out.stdout
