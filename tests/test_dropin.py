"""Runs the C++ drop-in test (tests/cpp/test_dropin.cpp): kcore::gpu::fastk_run
(the B200 path behind the reference's own signature and types) against the
reference library's peel_coreness and CPU fastk_run."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def test_cpp_dropin(gpu):
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/test_dropin not built (needs /root/reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
