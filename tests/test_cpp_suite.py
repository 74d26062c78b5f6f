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
