"""The reference-side C++ drop-in (integration/qbx3d/b200.hpp, shown in INTEGRATION.md)
compiled against the reference's own header /root/reference/proj/include/qbx3d/kernels.hpp
and linked with libqbxg.so and the reference's compiled kernels.cpp
(integration/Makefile; VERDICT r01 "next" #4): exception mapping without a device, and on
a B200 direct_sum_b200 == qbx::direct_sum, identical domain_error messages on a
coincidence, FmmB200::apply against qbx::direct_sum at far targets."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "integration", "_bin", "test_b200_wrapper")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "integration")], check=True)


def test_wrapper_builds_and_maps_errors():
    _build()
    if not os.path.exists(BIN):
        pytest.skip("reference headers absent and no prebuilt wrapper test")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert "FAIL" not in r.stdout, r.stdout
    assert r.returncode in (0, 77), (r.returncode, r.stdout, r.stderr)
    assert r.stdout.count("ok ") >= 2


@pytest.mark.gpu
def test_wrapper_on_device():
    if not os.path.exists(BIN):
        pytest.skip("wrapper test binary not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert "FAIL" not in r.stdout and r.stdout.count("ok ") >= 5, r.stdout
