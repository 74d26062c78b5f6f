"""Runs the C++ test binary (tests/cpp/*.cpp, built by `make tests`).

CPU part: wire codec, loopback + OS transports, doorbell, the GVM session
machine with a host test double, the client SDK, model + simulator.
GPU part ([gpu] cases): every payload kernel against the oracle through the
GVM (PS-1/PS-2, both data planes, loopback and forked OS clients),
PayloadRegistry::execute and the NativeVgpu baseline.
"""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "tests", "_bin", "vgpu-tests")


def _run(flag, timeout):
    p = subprocess.run([BIN, flag], cwd=REPO, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                       timeout=timeout, text=True)
    if p.returncode != 0:
        pytest.fail(p.stdout[-6000:])
    assert "0 failed" in p.stdout


def test_cpp_cpu_suite():
    _run("--exclude-gpu", 300)


@pytest.mark.gpu
def test_cpp_gpu_suite():
    _run("--only-gpu", 900)


# ---- drop-in proof: the reference's own unit tests against this library ----
# tests/_bin/ref-unit-tests is compiled in the build container from the
# UNMODIFIED /root/reference/proj/tests/test_{message,transport,model,device,
# daemon,client}.cpp with a doctest shim (oracle/Makefile.ref) and linked to
# libvgpu.so; the binary travels, the reference sources do not.
REF_BIN = os.path.join(REPO, "tests", "_bin", "ref-unit-tests")
# by design: the reference paces real-clock completions with sleeps
# (daemon.cpp:532-585); on B200 the real clock is the hardware's
REF_EXPECTED_DIFFERENT = ["real clock paces completion"]


def _ref_run(args, timeout):
    if not os.path.exists(REF_BIN):
        pytest.skip("ref-unit-tests not built (needs /root/reference at build time)")
    p = subprocess.run([REF_BIN] + args, cwd=REPO, stdout=subprocess.PIPE,
                       stderr=subprocess.STDOUT, timeout=timeout, text=True)
    if p.returncode != 0:
        pytest.fail(p.stdout[-6000:])
    assert "0 failed" in p.stdout


def test_reference_unit_tests_cpu_suites():
    _ref_run(["--file", "test_message", "--file", "test_transport", "--file", "test_model",
              "--file", "test_device"], 300)


@pytest.mark.gpu
def test_reference_unit_tests_all_on_b200():
    args = []
    for name in REF_EXPECTED_DIFFERENT:
        args += ["--skip", name]
    _ref_run(args, 600)
