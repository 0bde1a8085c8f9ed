"""Runs the C++ drop-in test (tests/cpp/test_dropin.cpp): kcore::gpu::fastk_run
(the B200 path behind the reference's own signature and types) against the
reference library's peel_coreness and CPU fastk_run."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")
SHIM = os.path.join(ROOT, "tests", "cpp", "test_shim")


def test_cpp_dropin(gpu):
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/test_dropin not built (needs /root/reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_cpp_link_time_shim(gpu):
    """The link-time drop-in (host/fastk_dropin_shim.cpp) linked INSTEAD of the
    reference's src/fastk.cpp: kcore::fastk_run itself runs on the B200 and the
    properties of the reference's tests/test_fastk.cpp (exact RunReport
    counters, hybrid tail, shadow replay) hold through it."""
    if not os.path.exists(SHIM):
        pytest.skip("tests/cpp/test_shim not built (needs /root/reference at build time)")
    r = subprocess.run([SHIM], capture_output=True, text=True, timeout=900)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
